"""Fused SP-attention AG-GEMM / GEMM-RS vs a torch fp32 reference."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [1, 2, 4])
def test_attn_ag_gemm_gemm_rs(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29700 + n}", os.path.join(ROOT, "tests", "mp_attn_check.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "ATTN_RESULT" in p.stdout


def test_attn_full_and_split_tail_tiles():
    """s = 8192, 640 QKV columns at TP = 4: 96 AG-GEMM pair tiles = one wave of 74
    full tiles + 22 tiles split into M = 128 pair tiles (split_last): both tile
    kinds against the fp32 reference, and the fused GEMM-RS bit-exact against the
    staging + reduce kernel."""
    n = 4
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29711", os.path.join(ROOT, "tests", "mp_attn_check.py")]
    env = dict(os.environ, MP_ATTN_S="8192", MP_ATTN_NQ="640")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "ATTN_RESULT" in p.stdout
