"""Multi-GPU (EP over NVLink) layer parity: spawns one process per GPU."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(n, env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29631", os.path.join(ROOT, "tests", "mp_layer_check.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "MP_RESULT" in p.stdout
    return p.stdout


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("cf", ["0", "1.0"])
def test_ep2_layer_parity(cf):
    _run(2, {"MP_CF": cf})


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("gate,comm", [("after_fc2_out", "fp8"), ("before_fc2_in", "fp8"), ("after_fc2_out", "bf16")])
def test_ep2_gate_order_fp8(gate, comm):
    _run(2, {"MP_CF": "1.0", "MP_GATE": gate, "MP_COMM": comm})


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs >= 4 GPUs")
def test_ep4_layer_parity():
    _run(4, {"MP_CF": "1.25"})
