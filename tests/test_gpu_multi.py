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


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("dedup", ["0", "1"])
def test_ep2_several_experts_per_token_on_a_rank(dedup):
    """k = 4 of E = 8 experts, 4 per rank: tokens reach a rank through several
    experts (the dispatch dedup path when enabled); >= 256 rows per expert, so
    CTA-pair tiles with M=128 tails."""
    env = {"MP_CF": "0", "MP_E": "8", "MP_K": "4", "MP_TR": "256"}
    if dedup == "0":
        env["MOE_NO_DISPATCH_DEDUP"] = "1"
    _run(2, env)


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs >= 4 GPUs")
def test_ep4_fine_grained_dedup():
    """DeepSeek-style routing at small scale: E = 32, k = 8, EP = 4, dedup on, drops."""
    _run(4, {"MP_CF": "1.25", "MP_E": "32", "MP_K": "8", "MP_TR": "256"})


def _run_full(n, cfg):
    env = dict(os.environ, MP_CFG=cfg)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29641", os.path.join(ROOT, "tests", "mp_fullshape_check.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    line = [ln for ln in p.stdout.splitlines() if "MP_FULL_RESULT" in ln]
    assert line, p.stdout[-2000:]
    print(line[0])


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs >= 4 GPUs")
@pytest.mark.parametrize("cfg", ["cfg2_mixtral", "cfg3_deepseek", "cfg5_fp8_zipf", "cfg5_fp8_zipf_cf1"])
def test_ep4_full_shape_parity(cfg):
    """BASELINE configs[1], [2], [4] at EP = 4, T_r = 4096 per rank: sampled
    fwd+bwd parity against the oracle, every rank's scatter map bit-exact."""
    _run_full(4, cfg)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_ep2_full_shape_parity_mixtral():
    _run_full(2, "cfg2_mixtral")


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("E,k,cf", [(8, 2, "0"), (8, 4, "1.25"), (32, 8, "0")])
def test_ep2_ag_rs_pattern(E, k, cf):
    """ep_pattern = ag_rs: in-kernel all-gather + local scatter, local expert
    rows pre-reduced per (token, rank) and reduce-scattered to the owner."""
    _run(2, {"MP_CF": cf, "MP_E": str(E), "MP_K": str(k), "MP_TR": "256", "MP_EP": "ag_rs"})


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs >= 4 GPUs")
def test_ep4_ag_rs_pattern():
    _run(4, {"MP_CF": "1.25", "MP_E": "32", "MP_K": "8", "MP_TR": "256", "MP_EP": "ag_rs"})


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs >= 4 GPUs")
def test_ep4_full_shape_parity_deepseek_ag_rs():
    env = dict(os.environ, MP_CFG="cfg3_deepseek", MP_EP="ag_rs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4",
           "--master-addr=127.0.0.1", "--master-port=29642", os.path.join(ROOT, "tests", "mp_fullshape_check.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "MP_FULL_RESULT" in p.stdout


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("ep", ["a2a", "ag_rs"])
def test_ep2_protocol_assertions(ep):
    """MOE_DEBUG_CHECKS=1 (device-side protocol assertions in place of the
    compute-sanitizer runs this pool does not allow): barrier epochs exact on
    every slot, every dispatch block landed exactly once, dedup rows once,
    all-gather chunks complete — over several steps, with drops and dedup."""
    _run(2, {"MP_CF": "1.25", "MP_E": "8", "MP_K": "4", "MP_TR": "256", "MP_EP": ep, "MOE_DEBUG_CHECKS": "1"})


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_ep2_timeout_status():
    """A peer that never arrives: the bounded flag waits give up and the status
    path returns MOE_ERR_TIMEOUT (no hang, no silent success)."""
    env = dict(os.environ, MOE_FLAG_TIMEOUT_MS="1500")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29651", os.path.join(ROOT, "tests", "mp_timeout_check.py")]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "TIMEOUT_RESULT ok" in p.stdout
