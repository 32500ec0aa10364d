"""BASELINE configs[0]: fp32 MoE layer forward (4096 tokens, hidden 1024,
ffn 2816, 8 experts top-2) against the fp32 CPU oracle.
Stated tolerance: relative L2 <= 1e-5 (bf16x6 tensor-core GEMMs: exact bf16
products of the three-piece split, fp32 accumulation; or the FFMA GEMMs with
MOE_F32_FFMA=1; vs the oracle's binary64 accumulation); routing bit-exact given
the same logits."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("gate_order", ["before_fc2_in", "after_fc2_out"])
def test_cfg1_fp32_forward_vs_oracle(gate_order):
    import pyoracle as P
    from paper_2505_11432_b200 import ops
    T, h, f, E, k = 4096, 1024, 2816, 8, 2
    rng = np.random.default_rng(1234)
    x = (rng.standard_normal((T, h)) * 0.5).astype(np.float32)
    w1 = (rng.standard_normal((E, 2 * f, h)) / np.sqrt(h)).astype(np.float32)
    w2 = (rng.standard_normal((E, h, f)) / np.sqrt(f)).astype(np.float32)
    wr = (rng.standard_normal((E, h)) / np.sqrt(h)).astype(np.float32)
    y, ex, g, lg, dr = ops.ffn_forward_f32(torch.from_numpy(x).cuda(), torch.from_numpy(w1).cuda(),
                                           torch.from_numpy(w2).cuda(), torch.from_numpy(wr).cuda(), k,
                                           gate_order=gate_order)
    torch.cuda.synchronize()
    olg, oex, og = P.orc_router_topk(x, wr, k)
    assert rel(lg.cpu().numpy(), olg) < 1e-5
    ex_np, g_np = ex.cpu().numpy(), g.cpu().numpy()
    sample = np.arange(0, T, 7)
    oy = P.orc_moe_forward(x, ex_np, g_np, dr.cpu().numpy(), w1, w2, tokens=sample,
                           gate_after=gate_order.startswith("after"))
    err = rel(y.cpu().numpy()[sample], oy)
    print("cfg1 fp32 rel err", err)
    assert err < 1e-5


def test_cfg1_fp32_injected_routing_with_golden_assignment():
    """The reference's own cfg1 routing (simulate_routing random, seed 11)."""
    import os
    import pyoracle as P
    from conftest import GOLDEN
    from paper_2505_11432_b200 import ops
    gd = np.load(os.path.join(GOLDEN, "routing_cfg1_random.npz"))
    T, E, k = int(gd["T"]), int(gd["E"]), int(gd["k"])
    h, f = 1024, 2816
    ex = gd["experts"].astype(np.int32).reshape(T, k)
    rng = np.random.default_rng(7)
    x = (rng.standard_normal((T, h)) * 0.5).astype(np.float32)
    w1 = (rng.standard_normal((E, 2 * f, h)) / np.sqrt(h)).astype(np.float32)
    w2 = (rng.standard_normal((E, h, f)) / np.sqrt(f)).astype(np.float32)
    gates = rng.random((T, k)).astype(np.float32)
    gates /= gates.sum(1, keepdims=True)
    y, _, _, _, dr = ops.ffn_forward_f32(torch.from_numpy(x).cuda(), torch.from_numpy(w1).cuda(),
                                         torch.from_numpy(w2).cuda(), None, k,
                                         experts=torch.from_numpy(ex).cuda(), gates=torch.from_numpy(gates).cuda())
    torch.cuda.synchronize()
    sample = np.arange(0, T, 5)
    oy = P.orc_moe_forward(x, ex, gates, np.zeros(T, np.uint8), w1, w2, tokens=sample)
    assert rel(y.cpu().numpy()[sample], oy) < 1e-5


def test_cfg1_fp32_ffma_path_same_tolerance():
    """The FFMA grouped-GEMM variant (MOE_F32_FFMA=1, read once per process) in a
    subprocess: same layer, same tolerance."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import pyoracle as P\nfrom paper_2505_11432_b200 import ops\n"
        "T,h,f,E,k=1024,1024,2816,8,2\nr=np.random.default_rng(3)\n"
        "x=(r.standard_normal((T,h))*0.5).astype(np.float32)\n"
        "w1=(r.standard_normal((E,2*f,h))/np.sqrt(h)).astype(np.float32)\n"
        "w2=(r.standard_normal((E,h,f))/np.sqrt(f)).astype(np.float32)\n"
        "wr=(r.standard_normal((E,h))/np.sqrt(h)).astype(np.float32)\n"
        "y,ex,g,lg,dr=ops.ffn_forward_f32(*(torch.from_numpy(a).cuda() for a in (x,w1,w2,wr)),k)\n"
        "s=np.arange(0,T,5)\noy=P.orc_moe_forward(x,ex.cpu().numpy(),g.cpu().numpy(),dr.cpu().numpy(),w1,w2,tokens=s)\n"
        "e=np.linalg.norm(y.cpu().numpy()[s]-oy)/np.linalg.norm(oy)\nprint('ERR',e)\nassert e<1e-5\n"
    ) % (root, os.path.join(root, "oracle"))
    p = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, MOE_F32_FFMA="1"),
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
