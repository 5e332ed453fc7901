"""Host-side check of the pair kernel's rotated wave order (DESIGN.md §12 item 1).

Compiles tests/native/tile_order_check.cu with nvcc for the HOST only (the schedule helpers in
csrc/kernels.h are __host__ __device__) and runs it: every shape's pair sequences must partition
the tiles exactly once without lengthening the busiest pair's list.  No GPU needed.
"""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not on PATH")
def test_pair_tile_order_partitions(tmp_path):
    exe = tmp_path / "tile_order_check"
    subprocess.run(["nvcc", "-std=c++17", "-O1", "-o", str(exe), os.path.join(HERE, "native", "tile_order_check.cu")],
                   check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("OK"), out.stdout
    # config 3 on 74 pairs: 592 first visits of an M block with the plain stride, 218 rotated, 102 matched
    assert "plain=592 rotated=218 matched=102" in out.stdout, out.stdout
