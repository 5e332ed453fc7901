"""World-N GPU test of the column-sharded path, N = every visible GPU.

Skipped on a box with fewer than 2 GPUs (this round's gpurun boxes have one; the world-1 runs of
the same plumbing are tests/test_gpu_dist.py).  torchrun starts one rank per GPU over NCCL on
127.0.0.1; every rank:
  * computes its column shard z_p = flashnorm_linear(a, W*[p]) (no collective: RMS is per token
    over K) and checks that ALL shards, all-gathered, are bit-identical to the
    unsharded 1-GPU result it computes locally (the invariant of §8(e));
  * gathers through the C ABI (flashnorm_comm_init + flashnorm_allgather_columns) and through
    torch.distributed + the library permute, both bit-identical to the unsharded result;
  * runs the epilogue-fused gather into every rank's symmetric-memory buffer
    (ColumnParallelFlashNorm.forward_fused_gather), bit-identical too, on two consecutive calls
    (the two alternating buffers).
"""
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
sys.path.insert(0, os.environ["FN_ROOT"])
import torch
import torch.distributed as dist
import paper_2407_09577_b200 as fn
from paper_2407_09577_b200.dist import ColumnParallelFlashNorm, shard_columns
from synth import device as SD

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
ok = True
for (M, K, N) in [(300, 512, 1024 * world), (16, 4096, 768 * world), (4096, 4096, 28672)]:
    a = SD.activations(3, M, K, dev, torch.bfloat16)
    W, g, b, c = SD.layer(3, N, K, dev, torch.bfloat16, with_b=True, with_c=True)
    Ws, cs = fn.fold_weights(W, g, b, c)
    full = fn.linear(a, Ws, cs, eps=1e-5)                      # the 1-GPU result, on every rank
    Wl, cl = shard_columns(Ws, cs, world, rank)
    zl = fn.linear(a, Wl.contiguous(), cl.contiguous(), eps=1e-5)
    parts = torch.empty((world, M, zl.shape[1]), dtype=zl.dtype, device=dev)
    dist.all_gather_into_tensor(parts.view(world * M, -1), zl)
    cat = torch.cat(list(parts), dim=1)
    ok &= torch.equal(cat.view(torch.int16), full.view(torch.int16))
    # C-ABI NCCL all-gather + permute
    uid = fn.comm_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
    dist.broadcast(t, 0)
    comm = fn.comm_init(bytes(t.cpu().tolist()), world, rank)
    assert fn.comm_count(comm) == world
    zc = fn.allgather_columns(zl, comm)
    torch.cuda.synchronize()
    ok &= torch.equal(zc.view(torch.int16), full.view(torch.int16))
    fn.comm_destroy(comm)
    layer = ColumnParallelFlashNorm(Wl.contiguous(), cl.contiguous(), world=world, rank=rank)
    zt = layer(a, gather=True)
    ok &= torch.equal(zt.view(torch.int16), full.view(torch.int16))
    for mc in ("auto", False):  # NVLS multimem.st when the group has a multicast mapping, and peer stores
        for _ in range(3):
            zf = layer.forward_fused_gather(a, eps=1e-5, multicast=mc)
            torch.cuda.synchronize()
            ok &= torch.equal(zf.view(torch.int16), full.view(torch.int16))
        if rank == 0:
            print("fused gather", mc, "->", layer.last_gather)
    del a, W, Ws, full, zl, parts, cat, zc, zt, layer
okt = torch.tensor([1 if ok else 0], device=dev)
dist.all_reduce(okt, op=dist.ReduceOp.MIN)
if rank == 0:
    print("MULTI_OK" if int(okt.item()) == 1 else "MULTI_FAIL", world)
dist.destroy_process_group()
'''


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs (world-1 plumbing: tests/test_gpu_dist.py)")
def test_column_shards_and_gathers_bit_exact_at_world_n():
    n = torch.cuda.device_count()
    env = dict(os.environ, FN_ROOT=ROOT)
    path = os.path.join(ROOT, "gpurun_out", "multi_script.py")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        f.write(SCRIPT)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                        "--master-addr=127.0.0.1", f"--master-port={_free_port()}", path],
                       env=env, capture_output=True, text=True, timeout=900)
    assert f"MULTI_OK {n}" in r.stdout, r.stdout[-3000:] + r.stderr[-5000:]
