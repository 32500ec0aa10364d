"""CPU suite: pin the oracle to the reference.

The oracle (oracle/moe_oracle.c, a C restatement) is checked bit-for-bit
against (a) the golden fixtures generated from the reference's own code and
(b) the reference library itself (oracle/_ref) when it is built here.
"""
import glob
import os

import numpy as np
import pytest

import pyoracle as P
from conftest import GOLDEN

CASES = sorted(c for c in glob.glob(os.path.join(GOLDEN, "routing_*.npz")) if "worked" not in c)


def _load(p):
    d = np.load(p)
    return {k: d[k] for k in d.files}


@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(c)[8:-4] for c in CASES])
def test_oracle_routing_matches_golden(path):
    g = _load(path)
    T, E, k, n, cf = int(g["T"]), int(g["E"]), int(g["k"]), int(g["n"]), float(g["cf"])
    ex = g["experts"].astype(np.int32).reshape(T, k)
    src = g["source_rank"].astype(np.int32)
    dr = P.orc_capacity_drop(ex, E, n, cf)
    assert (dr == g["dropped"]).all()
    bm = P.orc_balance_metrics(ex, dr, E, n)
    assert (bm["per_group_load"] == g["balance_load"]).all()
    assert bm["loss"] == float(g["balance_loss"])
    assert bm["capacity"] == int(g["balance_capacity"])
    assert bm["drop_rate"] == float(g["balance_drop_rate"])
    for r in range(n):
        m = P.orc_build_scatter_map(ex, src, dr, E, n, r)
        assert (m["row_map_in"] == g[f"r{r}_row_map_in"]).all()
        assert (m["out_expert"] == g[f"r{r}_out_expert"]).all()
        assert (m["out_source_rank"] == g[f"r{r}_out_source_rank"]).all()
        assert (m["per_expert_counts"] == g["per_expert_counts"]).all()
        for tr in (128, 3):
            t = P.orc_sort_tokens_for_tiles(m["out_expert"], m["out_source_rank"], tr)
            assert (t["expert"] == g[f"r{r}_t{tr}_expert"]).all()
            assert (t["begin"] == g[f"r{r}_t{tr}_begin"]).all()
            assert (t["end"] == g[f"r{r}_t{tr}_end"]).all()
            assert (t["rank_mask"].astype(np.uint64) == g[f"r{r}_t{tr}_mask"].astype(np.uint64)).all()


def test_oracle_worked_examples():
    g = _load(os.path.join(GOLDEN, "routing_worked_examples.npz"))
    ex = np.array([[1], [0], [0], [1]], np.int32)
    m = P.orc_build_scatter_map(ex, np.zeros(4, np.int32), np.zeros(4, np.uint8), 2, 2, 0)
    assert m["row_map_in"].tolist() == [1, 2] == g["ex4_row_map_in"].tolist()
    assert m["per_expert_counts"].tolist() == [2, 2] == g["ex4_counts"].tolist()
    ex = np.zeros((4, 1), np.int32)
    m = P.orc_build_scatter_map(ex, np.array([2, 0, 1, 0], np.int32), np.zeros(4, np.uint8), 3, 3, 0)
    assert m["out_source_rank"].tolist() == [0, 0, 1, 2]
    for tr in (2, 16):
        t = P.orc_sort_tokens_for_tiles(m["out_expert"], m["out_source_rank"], tr)
        assert t["rank_mask"].tolist() == g[f"ex2010_t{tr}_mask"].tolist()
    with pytest.raises(ValueError):
        P.orc_build_scatter_map(ex, np.zeros(4, np.int32), np.zeros(4, np.uint8), 2, 2, 2)


def test_oracle_numerics_matches_golden():
    g = _load(os.path.join(GOLDEN, "numerics.npz"))
    x = g["x"]
    for f in ("bf16", "fp8_e4m3", "fp32"):
        got = P.orc_round_to(f, x)
        want = g[f"round_{f}"]
        same = (got == want) | (np.isnan(got) & np.isnan(want))
        assert same.all(), f
    for gran in ("per_tensor", "per_token", "per_channel", "grouped"):
        c, s = P.orc_quantize(g["qx"], gran, "fp8_e4m3", 128)
        assert (c == g[f"q_{gran}_codes"]).all() and (s == g[f"q_{gran}_scales"]).all(), gran
    for kind in ("ring_bf16", "a2a_fp32"):
        assert (P.orc_emulate_reduce(g["rv"], kind) == g[f"reduce_{kind}"]).all()
    assert P.orc_emulate_reduce(np.array([[1024.0], [1.0], [1.0]]), "ring_bf16")[0] == 1025.0
    assert P.orc_emulate_reduce(np.array([[1024.0], [1.0], [1.0]]), "a2a_fp32")[0] == 1026.0


def test_worked_rounding_values():
    """test_numerics.cpp:29-55 worked values."""
    r = P.orc_round_to
    assert r("fp8_e4m3", [1.0])[0] == 1.0
    assert r("fp8_e4m3", [500.0])[0] == 448.0
    assert r("fp8_e4m3", [-500.0])[0] == -448.0
    assert r("fp8_e4m3", [449.0])[0] == 448.0
    assert r("fp8_e4m3", [465.0])[0] == 448.0
    assert r("fp8_e4m3", [1.0625])[0] == 1.0
    assert r("bf16", [1e39])[0] == np.inf
    assert r("bf16", [1.0 + 1.0 / 256.0])[0] == 1.0
    assert r("bf16", [1.0 + 3.0 / 256.0])[0] == 1.0 + 2.0 / 128.0


@pytest.mark.skipif(not P.ref_available(), reason="reference build (oracle/_ref) not present")
def test_oracle_vs_reference_live():
    """Fresh random assignments through the reference and the oracle."""
    rng = np.random.default_rng(5)
    for trial in range(20):
        T = int(rng.integers(1, 600))
        n = int(rng.choice([1, 2, 4, 8]))
        E = n * int(rng.integers(1, 5))
        k = int(rng.integers(1, min(E, 4) + 1))
        mode = ["uniform", "random", "skewed"][trial % 3]
        cf = float(rng.choice([0.5, 1.0, 1.25, 1e9]))
        ex, src, dr = P.ref_simulate_routing(T, E, k, mode, int(rng.integers(0, 1 << 30)), 1.2, cf, n)
        assert (P.orc_capacity_drop(ex, E, n, cf) == dr).all()
        for r in range(n):
            a = P.ref_build_scatter_map(ex, src, dr, E, n, r)
            b = P.orc_build_scatter_map(ex, src, dr, E, n, r)
            for key in ("row_map_in", "per_expert_counts", "out_expert", "out_source_rank"):
                assert (a[key] == b[key]).all()
            for tr in (1, 5, 128):
                ta = P.ref_sort_tokens_for_tiles(ex, src, dr, E, n, r, tr)
                tb = P.orc_sort_tokens_for_tiles(b["out_expert"], b["out_source_rank"], tr)
                for key in ("expert", "begin", "end", "rank_mask"):
                    assert (ta[key] == tb[key]).all()
    x = np.ldexp(rng.standard_normal(20000), rng.integers(-150, 136, 20000))
    for f in ("bf16", "fp8_e4m3", "fp32"):
        assert (P.ref_round_to(f, x) == P.orc_round_to(f, x)).all()


def test_dense_oracle_self_consistency():
    """Finite-difference check of the dense oracle's backward (small shape)."""
    rng = np.random.default_rng(1)
    T, h, f, E, k = 6, 16, 8, 4, 2
    x = rng.standard_normal((T, h)).astype(np.float32)
    w1 = (rng.standard_normal((E, 2 * f, h)) * 0.3).astype(np.float32)
    w2 = (rng.standard_normal((E, h, f)) * 0.3).astype(np.float32)
    wr = (rng.standard_normal((E, h)) * 0.3).astype(np.float32)
    dy = rng.standard_normal((T, h)).astype(np.float32)
    lg, ex, g = P.orc_router_topk(x, wr, k)
    dr = np.zeros(T, np.uint8)
    b = P.orc_moe_backward(x, dy, ex, g, lg, dr, w1, w2, wr)

    def loss(w1_):
        y = P.orc_moe_forward(x, ex, g, dr, w1_, w2)
        return float((y.astype(np.float64) * dy).sum())
    eps = 1e-3
    for (e, j, c) in ((0, 1, 2), (1, f + 3, 5), (3, 2 * f - 1, h - 1)):
        if not (ex == e).any():
            continue
        wp, wm = w1.copy(), w1.copy()
        wp[e, j, c] += eps
        wm[e, j, c] -= eps
        fd = (loss(wp) - loss(wm)) / (2 * eps)
        assert abs(fd - b["dw1"][e, j, c]) < 2e-2 * max(1.0, abs(fd))


@pytest.mark.parametrize("gate_after", [False, True])
def test_bf16_sampled_restatement_matches_dense_oracle(gate_after):
    """The bf16-input sampled oracle (full-shape parity tests) agrees with the
    fp32 dense oracle on rows, dgates and the sampled weight-gradient columns."""
    import torch
    T, h, f, E, k = 48, 64, 96, 4, 2
    g = torch.Generator().manual_seed(3)
    x = (torch.randn(T, h, generator=g) * 0.5).bfloat16()
    dy = (torch.randn(T, h, generator=g) * 0.1).bfloat16()
    w1 = (torch.randn(E, 2 * f, h, generator=g) / h ** 0.5).bfloat16()
    w2 = (torch.randn(E, h, f, generator=g) / f ** 0.5).bfloat16()
    wr = (torch.randn(E, h, generator=g) / h ** 0.5).bfloat16()
    xf, dyf, w1f, w2f, wrf = (t.float().numpy() for t in (x, dy, w1, w2, wr))
    lg, ex, gt = P.orc_router_topk(xf, wrf, k)
    dr = np.zeros(T, np.uint8)
    dr[5] = 1
    toks = np.array([0, 3, 5, 17, 47])
    r = P.orc_moe_rows_bf16(x, dy, ex, gt, dr, w1, w2, wr, toks, gate_after=gate_after)
    oy = P.orc_moe_forward(xf, ex, gt, dr, w1f, w2f, tokens=toks, gate_after=gate_after)
    ob = P.orc_moe_backward(xf, dyf, ex, gt, lg, dr, w1f, w2f, wrf, gate_after=gate_after)
    np.testing.assert_allclose(r["y"], oy, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(r["dx"], ob["dx"][toks], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(r["dgates"], ob["dgates"][toks], rtol=1e-4, atol=1e-6)
    cols = np.array([0, 7, f - 1])
    dw1, dw2 = P.orc_moe_wgrad_cols_bf16(x, dy, ex, gt, dr, w1, w2, cols, gate_after=gate_after)
    np.testing.assert_allclose(dw1[:, :, 0], ob["dw1"][:, cols], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(dw1[:, :, 1], ob["dw1"][:, f + cols], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(dw2, ob["dw2"][:, :, cols].transpose(0, 2, 1), rtol=1e-4, atol=1e-6)
    dwr = P.orc_router_wgrad_from_dgates(xf, ex, gt, ob["dgates"], dr, E)
    np.testing.assert_allclose(dwr, ob["dwr"], rtol=1e-4, atol=1e-6)


def test_numpy_blas_dense_restatement_matches_c_oracle():
    """The numpy/BLAS dense restatement (bench.py's full-shape CPU baseline)
    computes the same layer as the C oracle."""
    rng = np.random.default_rng(4)
    T, h, f, E, k = 40, 64, 96, 4, 2
    x = rng.standard_normal((T, h)).astype(np.float32) * 0.5
    dy = rng.standard_normal((T, h)).astype(np.float32) * 0.1
    w1 = rng.standard_normal((E, 2 * f, h)).astype(np.float32) / 8
    w2 = rng.standard_normal((E, h, f)).astype(np.float32) / 10
    wr = rng.standard_normal((E, h)).astype(np.float32) / 8
    lg, ex, gt = P.orc_router_topk(x, wr, k)
    nlg, nex, ngt = P.np_router_topk(x, wr, k)
    assert (nex == ex).all()
    np.testing.assert_allclose(ngt, gt, rtol=1e-5)
    dr = np.zeros(T, np.uint8)
    y, dx, dg, (dw1, dw2, dwr) = P.np_moe_fwd_bwd(x, dy, wr, w1, w2, k, ex, gt, dr)
    oy = P.orc_moe_forward(x, ex, gt, dr, w1, w2)
    ob = P.orc_moe_backward(x, dy, ex, gt, lg, dr, w1, w2, wr)
    for a, b in ((y, oy), (dx, ob["dx"]), (dg, ob["dgates"]), (dw1, ob["dw1"]), (dw2, ob["dw2"]), (dwr, ob["dwr"])):
        np.testing.assert_allclose(a, b, rtol=2e-4, atol=2e-5)
