"""Generate tests/golden/ fixtures by running the REFERENCE's own code
(oracle/_ref/libmoeplan_ref.so, compiled from /root/reference/proj/core/src).

TEST INFRASTRUCTURE ONLY. Run in the build container (where /root/reference
exists):  python oracle/gen_golden.py
The fixtures are committed so tests on the GPU box (no /root/reference) can
pin the oracle and the CUDA path to the reference's outputs.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import pyoracle as P  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

# (name, T, E, k, mode, seed, zipf_s, cf, n) — the BASELINE.json routing shapes
# plus the reference tests' own parameter sets.
ROUTING_CASES = [
    ("cfg1_random", 4096, 8, 2, "random", 11, 1.0, 1e9, 1),
    ("cfg2_random_n8", 32768, 8, 2, "random", 11, 1.0, 1e9, 8),
    ("cfg2_refgeom_n8", 4096, 8, 2, "random", 11, 1.0, 1e9, 8),
    ("cfg3_random_n8", 32768, 256, 8, "random", 11, 1.0, 1e9, 8),
    ("cfg5_zipf_nodrop_n8", 32768, 8, 2, "skewed", 11, 1.2, 1e9, 8),
    ("cfg5_zipf_cf1_n8", 32768, 8, 2, "skewed", 11, 1.2, 1.0, 8),
    # test_routing.cpp parameter sets
    ("t_uniform_64", 64, 8, 2, "uniform", 0, 1.0, 1.0, 8),
    ("t_random_256_cf125", 256, 16, 2, "random", 42, 1.0, 1.25, 8),
    ("t_random_200_k4", 200, 8, 4, "random", 3, 1.0, 10.0, 8),
    ("t_skewed_4096_k1", 4096, 8, 1, "skewed", 11, 1.2, 1.0, 8),
    ("t_skewed_512_s11", 512, 16, 2, "skewed", 7, 1.1, 1.0, 8),
    ("t_random_128_n4", 128, 8, 2, "random", 5, 1.0, 1.0, 4),
    ("t_random_96_n4", 96, 8, 2, "random", 9, 1.0, 2.0, 4),
    ("t_skewed_128_s13", 128, 8, 2, "skewed", 21, 1.3, 1.0, 8),
]

TILE_ROWS = (128, 3)


def routing_fixture(name, T, E, k, mode, seed, zipf_s, cf, n):
    ex, src, dr = P.ref_simulate_routing(T, E, k, mode, seed, zipf_s, cf, n)
    d = dict(T=T, E=E, k=k, n=n, cf=cf, seed=seed, zipf_s=zipf_s, mode=mode,
             experts=ex.astype(np.int16 if E < 32768 else np.int32), source_rank=src.astype(np.int8),
             dropped=dr)
    bm = P.ref_balance_metrics(ex, src, dr, E, n)
    d.update(balance_load=bm["per_group_load"], balance_loss=bm["loss"],
             balance_capacity=bm["capacity"], balance_drop_rate=bm["drop_rate"])
    for r in range(n):
        m = P.ref_build_scatter_map(ex, src, dr, E, n, r)
        d[f"r{r}_row_map_in"] = m["row_map_in"].astype(np.int32)
        d[f"r{r}_out_expert"] = m["out_expert"].astype(np.int16)
        d[f"r{r}_out_source_rank"] = m["out_source_rank"].astype(np.int8)
        assert (m["row_map_out"] == np.arange(m["rows"])).all()
        assert (m["inverse_map"] == m["row_map_in"]).all()
        if r == 0:
            d["per_expert_counts"] = m["per_expert_counts"].astype(np.int32)
        for tr in TILE_ROWS:
            t = P.ref_sort_tokens_for_tiles(ex, src, dr, E, n, r, tr)
            d[f"r{r}_t{tr}_expert"] = t["expert"].astype(np.int16)
            d[f"r{r}_t{tr}_begin"] = t["begin"].astype(np.int32)
            d[f"r{r}_t{tr}_end"] = t["end"].astype(np.int32)
            d[f"r{r}_t{tr}_mask"] = t["rank_mask"].astype(np.uint16)
    np.savez_compressed(os.path.join(OUT, f"routing_{name}.npz"), **d)


def worked_examples():
    """test_routing.cpp:114-128 and :168-182, run through the reference."""
    out = {}
    ex = np.array([[1], [0], [0], [1]], np.int32)
    src = np.zeros(4, np.int32)
    dr = np.zeros(4, np.uint8)
    m = P.ref_build_scatter_map(ex, src, dr, 2, 2, 0, n_groups=2)
    out["ex4_row_map_in"] = m["row_map_in"]
    out["ex4_counts"] = m["per_expert_counts"]
    ex = np.zeros((4, 1), np.int32)
    src = np.array([2, 0, 1, 0], np.int32)
    m = P.ref_build_scatter_map(ex, src, dr, 3, 3, 0, n_groups=3)
    out["ex2010_row_map_in"] = m["row_map_in"]
    out["ex2010_out_source_rank"] = m["out_source_rank"]
    for tr in (2, 16):
        t = P.ref_sort_tokens_for_tiles(ex, src, dr, 3, 3, 0, tr, n_groups=3)
        out[f"ex2010_t{tr}_mask"] = t["rank_mask"]
        out[f"ex2010_t{tr}_begin"] = t["begin"]
        out[f"ex2010_t{tr}_end"] = t["end"]
    np.savez_compressed(os.path.join(OUT, "routing_worked_examples.npz"), **out)


def numerics_fixture():
    rng = np.random.default_rng(123)
    x = np.ldexp(rng.standard_normal(30000), rng.integers(-150, 136, 30000))
    special = np.array([1.0, 448.0, 500.0, -500.0, 449.0, 465.0, 1.0625, 1e39, 0.0,
                        1.0 + 1.0 / 256.0, 1.0 + 3.0 / 256.0, np.inf, -np.inf, 2.0 ** -9,
                        2.0 ** -10, 3 * 2.0 ** -10, 1.5 * 2.0 ** -133])
    x = np.concatenate([special, x])
    d = dict(x=x)
    for f in ("bf16", "fp8_e4m3", "fp32"):
        d[f"round_{f}"] = P.ref_round_to(f, x)
    q = rng.standard_normal((16, 300)) * np.exp(rng.standard_normal((16, 1)) * 2)
    q[3] = 0.0
    d["qx"] = q
    for g in ("per_tensor", "per_token", "per_channel", "grouped"):
        c, s = P.ref_quantize(q, g, "fp8_e4m3", 128)
        d[f"q_{g}_codes"], d[f"q_{g}_scales"] = c, s
    v = rng.standard_normal((8, 2048))
    d["rv"] = v
    for kind in ("ring_bf16", "a2a_fp32"):
        d[f"reduce_{kind}"] = P.ref_emulate_reduce(v, kind)
    d["reduce_1024_ring"] = P.ref_emulate_reduce(np.array([[1024.0], [1.0], [1.0]]), "ring_bf16")
    d["reduce_1024_wide"] = P.ref_emulate_reduce(np.array([[1024.0], [1.0], [1.0]]), "a2a_fp32")
    np.savez_compressed(os.path.join(OUT, "numerics.npz"), **d)


def main():
    os.makedirs(OUT, exist_ok=True)
    if not P.ref_available():
        P.build()
    worked_examples()
    numerics_fixture()
    for case in ROUTING_CASES:
        routing_fixture(*case)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
