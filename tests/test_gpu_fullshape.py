"""Full-shape parity of the MoE layer on one GPU at the benchmarked
configurations (BASELINE.json configs[1], [2], [4]; T_r = 4096 tokens, fwd+bwd).
Sampling and tolerances: tests/fullshape_common.py."""
import numpy as np
import pytest
import torch

from fullshape_common import CONFIGS, check_routing, dense_errors, make_inputs, sample, tolerance, wgrad_cols, zipf_routing

pytestmark = pytest.mark.gpu
T = 4096


@pytest.mark.parametrize("name", [c for c in CONFIGS if "cf" not in CONFIGS[c]])
def test_full_shape_sampled_parity(name):
    import pyoracle as P
    from conftest import GOLDEN
    from paper_2505_11432_b200.layer import MoELayer
    c = CONFIGS[name]
    h, f, E, k = c["h"], c["f"], c["E"], c["k"]
    w1, w2, wr, x, dy = make_inputs(c, T)
    L = MoELayer(T, h, f, E, k, route_mode="injected" if c["route"] == "zipf" else "learned",
                 gate_order=c["gate"], comm_format=c["comm"])
    L.set_weights(w1, w2, wr)
    if c["route"] == "zipf":
        ex_in, gt_in = zipf_routing(GOLDEN, T, k)
        L.set_routing(torch.from_numpy(ex_in).cuda(), torch.from_numpy(gt_in).cuda())
    y = L.forward(x)
    dx, dw1, dw2, dwr = L.backward(dy)
    L.status()
    r = L.routing()
    ex, gt, dr, dg, lg = (r[q].cpu().numpy() for q in ("experts", "gates", "dropped", "dgates", "logits"))
    assert dr.sum() == 0  # no capacity factor: nothing dropped
    if c["route"] == "zipf":
        assert (ex == ex_in).all() and np.array_equal(gt, gt_in)
    toks, cols = sample(T, f)
    errs = {}
    lerr, maps = check_routing(P, c, ex, gt, dr, lg, toks, x, wr, 1, T)
    if lerr is not None:
        errs["logits"] = lerr
        assert lerr < 1e-4, errs
    assert (r["row_map_in"].cpu().numpy() == maps[0]["row_map_in"]).all()
    assert (r["per_expert_counts"].cpu().numpy() == maps[0]["per_expert_counts"]).all()
    g1, g2 = wgrad_cols(dw1, dw2, cols, f)
    errs.update(dense_errors(P, c, ex, gt, dr, dg, toks, cols, x, dy, w1, w2, wr,
                             y.float().cpu().numpy()[toks], dx.float().cpu().numpy()[toks],
                             g1.cpu().numpy(), g2.cpu().numpy(), dwr.cpu().numpy()))
    print(name, {kk: f"{v:.2e}" for kk, v in errs.items()})
    bad = {kk: v for kk, v in errs.items() if kk != "logits" and not v < tolerance(c, kk)}
    assert not bad, (name, errs)
