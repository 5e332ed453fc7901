"""The fused-gather column-parallel path through torch symmetric memory + NCCL, on the ONE GPU
this round has (world_size = 1 process group: the rendezvous, peer-buffer and device-barrier
plumbing runs for real; the multi-GPU NVLink stores are the same st.global instructions the
several-destination test in test_gpu_parity.py exercises locally)."""
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import torch
import torch.distributed as dist
import paper_2407_09577_b200 as fn
from paper_2407_09577_b200.dist import ColumnParallelFlashNorm
from synth import device as SD
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
M, K, N = 300, 512, 1024
a = SD.activations(3, M, K, "cuda", torch.bfloat16)
W, g, b, c = SD.layer(3, N, K, "cuda", torch.bfloat16, with_b=True, with_c=True)
Ws, cs = fn.fold_weights(W, g, b, c)
layer = ColumnParallelFlashNorm.from_full(Ws, cs)
ref = fn.linear(a, Ws, cs, eps=1e-5)
for _ in range(3):
    out = layer.forward_fused_gather(a, eps=1e-5)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16)), "fused gather differs"
try:
    layer.forward_fused_gather(a, eps=1e-5, multicast=True)
    assert layer.last_gather == "multicast"
    print("MULTICAST_AVAILABLE")
except RuntimeError as e:
    assert "no NVLS multicast mapping" in str(e)
g2 = layer(a, gather=True)
assert torch.equal(g2.view(torch.int16), ref.view(torch.int16))
dist.destroy_process_group()
print("FUSED_GATHER_OK")
'''


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_fused_gather_symmetric_memory_world1():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=300)
    assert "FUSED_GATHER_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


SCRIPT_ABI = r'''
import sys
sys.path.insert(0, sys.argv[1])
import torch
import paper_2407_09577_b200 as fn
from synth import device as SD
torch.cuda.set_device(0)
uid = fn.comm_unique_id()
comm = fn.comm_init(uid, 1, 0)
a = SD.activations(4, 200, 512, "cuda", torch.bfloat16)
W, g, _, _ = SD.layer(4, 512, 512, "cuda", torch.bfloat16)
Ws, cs = fn.fold_weights(W, g)
zl = fn.linear(a, Ws, cs)
z = fn.allgather_columns(zl, comm, 1)
torch.cuda.synchronize()
assert torch.equal(z.view(torch.int16), zl.view(torch.int16))
fn.comm_destroy(comm)
print("NCCL_ABI_OK")
'''


def test_nccl_allgather_through_the_c_abi_world1():
    """flashnorm_comm_unique_id / comm_init / allgather_columns / comm_destroy with one rank:
    NCCL loaded by the library (dlopen), the all-gather + permute returns the shard itself."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, "-c", SCRIPT_ABI, ROOT], capture_output=True, text=True, timeout=300)
    assert "NCCL_ABI_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
