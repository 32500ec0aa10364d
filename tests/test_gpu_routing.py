"""GPU parity of K1/K2 routing kernels against the REFERENCE's own outputs
(tests/golden, produced by oracle/_ref from /root/reference sources) and the
CPU oracle. Bit-exact for every integer output."""
import glob
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CASES = sorted(glob.glob(os.path.join(GOLDEN, "routing_*.npz")))
CASES = [c for c in CASES if "worked" not in c]


def _load(path):
    d = np.load(path)
    return {k: d[k] for k in d.files}


@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(c)[8:-4] for c in CASES])
def test_routing_maps_bit_exact(path):
    from paper_2505_11432_b200 import routing as R
    g = _load(path)
    T, E, k, n, cf = int(g["T"]), int(g["E"]), int(g["k"]), int(g["n"]), float(g["cf"])
    ex = g["experts"].astype(np.int32).reshape(T, k)
    src = g["source_rank"].astype(np.int32)
    a = R.RoutingAssignment.from_host(E, k, n, ex, src)
    # capacity drop on the GPU reproduces the reference's drop flags
    dropped = R.capacity_drop(a, cf).cpu().numpy()
    assert (dropped == g["dropped"]).all()
    bm = R.balance_metrics(a, n)
    assert (bm.per_group_load.cpu().numpy() == g["balance_load"]).all()
    assert bm.balance_loss_value == float(g["balance_loss"])
    assert bm.capacity == int(g["balance_capacity"])
    assert bm.drop_rate == float(g["balance_drop_rate"])
    for r in range(n):
        m = R.build_scatter_map(a, n, r)
        assert m.rows == len(g[f"r{r}_row_map_in"])
        assert (m.row_map_in.cpu().numpy() == g[f"r{r}_row_map_in"]).all()
        assert (m.out_expert.cpu().numpy() == g[f"r{r}_out_expert"]).all()
        assert (m.out_source_rank.cpu().numpy() == g[f"r{r}_out_source_rank"]).all()
        assert (m.per_expert_counts.cpu().numpy() == g["per_expert_counts"]).all()
        for tr in (128, 3):
            lay = R.sort_tokens_for_tiles(m, a, tr)
            assert (lay.expert.cpu().numpy() == g[f"r{r}_t{tr}_expert"]).all()
            assert (lay.row_begin.cpu().numpy() == g[f"r{r}_t{tr}_begin"]).all()
            assert (lay.row_end.cpu().numpy() == g[f"r{r}_t{tr}_end"]).all()
            assert (lay.rank_mask.cpu().numpy().astype(np.uint64) == g[f"r{r}_t{tr}_mask"].astype(np.uint64)).all()


def test_worked_examples():
    """test_routing.cpp:114-128 and :168-182 through the GPU path."""
    from paper_2505_11432_b200 import routing as R
    from paper_2505_11432_b200 import DomainError
    g = _load(os.path.join(GOLDEN, "routing_worked_examples.npz"))
    a = R.RoutingAssignment.from_host(2, 1, 2, [1, 0, 0, 1], [0, 0, 0, 0])
    m = R.build_scatter_map(a, 2, 0)
    assert m.rows == 2
    assert m.row_map_in.cpu().tolist() == [1, 2] == g["ex4_row_map_in"].tolist()
    assert m.row_map_out.cpu().tolist() == [0, 1]
    assert m.inverse_map.cpu().tolist() == [1, 2]
    assert m.per_expert_counts.cpu().tolist() == [2, 2]
    b = R.RoutingAssignment.from_host(2, 1, 2, [1, 1, 1, 1], [0, 0, 0, 0])
    assert R.build_scatter_map(b, 2, 0).rows == 0
    with pytest.raises(DomainError):
        R.build_scatter_map(a, 2, 2)
    a = R.RoutingAssignment.from_host(3, 1, 3, [0, 0, 0, 0], [2, 0, 1, 0])
    m = R.build_scatter_map(a, 3, 0)
    assert m.rows == 4
    assert m.out_source_rank.cpu().tolist() == [0, 0, 1, 2]
    lay = R.sort_tokens_for_tiles(m, a, 2)
    assert len(lay) == 2
    assert lay.dependent_ranks(0) == [0]
    assert lay.dependent_ranks(1) == [1, 2]
    one = R.sort_tokens_for_tiles(m, a, 16)
    assert len(one) == 1 and one.dependent_ranks(0) == [0, 1, 2]


def test_empty_and_invalid():
    from paper_2505_11432_b200 import routing as R
    from paper_2505_11432_b200 import DomainError
    a = R.RoutingAssignment.from_host(8, 2, 8, np.zeros((0, 2), np.int32), np.zeros(0, np.int32))
    m = R.build_scatter_map(a, 8, 3)
    assert m.rows == 0 and int(m.per_expert_counts.sum()) == 0
    with pytest.raises(DomainError):
        R.build_scatter_map(R.RoutingAssignment.from_host(5, 1, 1, [0], [0]), 2, 0)
    with pytest.raises(DomainError):
        R.capacity_drop(R.RoutingAssignment.from_host(8, 2, 8, [[0, 1]], [0]), 0.0)


def test_topk_from_logits_bit_exact():
    """Selection is bit-exact given identical logits (ties -> lower id)."""
    from paper_2505_11432_b200 import routing as R
    import pyoracle as P
    rng = np.random.default_rng(0)
    for E, k in ((8, 2), (256, 8), (16, 4)):
        lg = rng.standard_normal((2048, E)).astype(np.float32)
        lg[::7, 1] = lg[::7, 0]                     # forced ties
        lg[::11] = np.round(lg[::11] * 4) / 4       # many ties
        ex, gates = R.topk_from_logits(torch.from_numpy(lg).cuda(), k)
        # oracle selection on the same logits
        want = np.argsort(-lg, axis=1, kind="stable")[:, :k]
        assert (ex.cpu().numpy() == want).all()
        sel = np.take_along_axis(lg.astype(np.float64), want, 1)
        ref = np.exp(sel - sel[:, :1]); ref /= ref.sum(1, keepdims=True)
        np.testing.assert_allclose(gates.cpu().numpy(), ref, rtol=1e-6, atol=1e-7)


def test_router_topk_vs_oracle():
    from paper_2505_11432_b200 import routing as R
    import pyoracle as P
    torch.manual_seed(0)
    T, h, E, k = 512, 1024, 8, 2
    x = (torch.randn(T, h) * 0.5).bfloat16()
    wr = (torch.randn(E, h) / h ** 0.5).bfloat16()
    lg, ex, g = R.router_topk(x.cuda(), wr.cuda(), k)
    olg, oex, og = P.orc_router_topk(x.float().numpy(), wr.float().numpy(), k)
    np.testing.assert_allclose(lg.cpu().numpy(), olg, rtol=1e-4, atol=1e-4)
    # selection agrees wherever the oracle's top-k margin exceeds the fp32 noise
    s = np.sort(olg, 1)[:, ::-1]
    clear = (s[:, k - 1] - s[:, k]) > 1e-3
    assert (ex.cpu().numpy()[clear] == oex[clear]).all()
    np.testing.assert_allclose(g.cpu().numpy()[clear], og[clear], rtol=1e-4, atol=1e-5)


def test_reference_test_routing_against_gpu_adapter():
    """The reference's own tests/test_routing.cpp, compiled unmodified against
    the drop-in adapter (libmoeplan_compat.so -> sm_100a kernels)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "oracle", "_ref", "ref_test_routing_on_gpu")
    if not os.path.exists(exe):
        pytest.skip("reference test binary not built (needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(p.stdout[-2000:])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert "0 failed" in p.stdout
