"""The reference's own hot-path integer / numerics code (oracle/_ref, compiled
from routing.cpp + numerics.cpp; single-threaded as shipped) timed at full
shape on the host, beside this repo's device kernels for the same work
(the reference's bench does the same list,
bench_moeplan.cpp:128-170):
  - build_scatter_map x n ranks       (cfg2 geometry: T = 32768, n = 8)
  - sort_tokens_for_tiles(128) x n ranks
  - balance_metrics
  - quantize(per_token, E4M3)         4096 x 4096
  - emulate_reduce(a2a_fp32)          8 ranks x 4096 x 4096
simulate_routing is the input generator and is timed separately (host only).
The device side goes through the C ABI with device-resident inputs and
outputs (moe_permute / moe_tile_layout / moe_balance_counts / moe_quantize /
moe_emulate_reduce; binary64, bit-exact), timed with CUDA events.
TEST / BASELINE INFRASTRUCTURE: bench.py's cpu_baseline leg only.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def _best(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1000.0 * float(np.median(ts))


def cpu_integer_path(T=32768, E=8, k=2, n=8, rows=4096, cols=4096, ranks=8, reps=3):
    import pyoracle as P
    use_ref = P.ref_available()
    t0 = time.perf_counter()
    ex, src, dr = (P.ref_simulate_routing(T, E, k, "random", 11, n_groups=n) if use_ref else (None, None, None))
    sim_ms = 1000.0 * (time.perf_counter() - t0)
    if not use_ref:
        rng = np.random.default_rng(11)
        ex = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
        src = (np.arange(T) * n // T).astype(np.int32)
        dr = np.zeros(T, np.uint8)
    res = {"kind": "reference" if use_ref else "port", "threads": 1,
           "simulate_routing_ms": round(sim_ms, 3)}
    rng = np.random.default_rng(1)
    xq = rng.standard_normal((rows, cols))
    vec = rng.standard_normal((ranks, rows * cols))
    if use_ref:
        # timed inside the reference library: value types built once, outside
        r_ms = P.ref_time_routing(ex, src, dr, E, n, 128, reps)
        q_ms = P.ref_time_numerics(xq, vec)
        res.update(build_scatter_map_x_n_ms=round(float(r_ms[0]), 3),
                   sort_tokens_for_tiles_x_n_ms=round(float(r_ms[1]), 3),
                   balance_metrics_ms=round(float(r_ms[2]), 3), quantize_per_token_e4m3_ms=round(float(q_ms[0]), 3),
                   emulate_reduce_a2a_fp32_ms=round(float(q_ms[1]), 3))
    else:
        res["build_scatter_map_x_n_ms"] = round(_best(
            lambda: [P.orc_build_scatter_map(ex, src, dr, E, n, r) for r in range(n)], reps), 3)
        res["quantize_per_token_e4m3_ms"] = round(_best(lambda: P.orc_quantize(xq, "per_token", "fp8_e4m3"), 1), 3)
        res["emulate_reduce_a2a_fp32_ms"] = round(_best(lambda: P.orc_emulate_reduce(vec, "a2a_fp32"), 1), 3)
    res["total_ms"] = round(sum(v for kk, v in res.items() if kk.endswith("_ms") and kk != "simulate_routing_ms"), 3)
    res["shapes"] = {"T": T, "E": E, "k": k, "n": n, "quantize": [rows, cols], "emulate_reduce": [ranks, rows * cols]}
    return res, (ex, src, dr, xq, vec)


def gpu_integer_path(inputs, T=32768, E=8, k=2, n=8, rows=4096, cols=4096, ranks=8, reps=10):
    import torch
    from paper_2505_11432_b200 import lib
    L = lib()
    L.moe_permute_workspace_size.restype = C.c_size_t
    L.moe_quantize_workspace_size.restype = C.c_size_t
    L.moe_quantize_num_blocks.restype = C.c_int64
    ex, src, dr, xq, vec = inputs
    dev = "cuda"
    i64 = C.c_int64
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    d_ex = torch.from_numpy(np.ascontiguousarray(ex, np.int32)).to(dev)
    d_src = torch.from_numpy(np.ascontiguousarray(src, np.int32)).to(dev)
    d_dr = torch.from_numpy(np.ascontiguousarray(dr, np.uint8)).to(dev)
    el = E // n
    cap = T * k
    ws = torch.empty(int(L.moe_permute_workspace_size(i64(T), i64(E), i64(k), i64(n))), dtype=torch.uint8, device=dev)
    rmi, oe, osr = (torch.empty(cap, dtype=torch.int32, device=dev) for _ in range(3))
    cnt = torch.empty(E, dtype=torch.int32, device=dev)
    eoff = torch.empty(el + 1, dtype=torch.int32, device=dev)
    nrows = torch.empty(1, dtype=torch.int32, device=dev)
    te, tb, tend = (torch.empty(cap + el, dtype=torch.int32, device=dev) for _ in range(3))
    tm = torch.empty(cap + el, dtype=torch.int64, device=dev)
    nt = torch.empty(1, dtype=torch.int32, device=dev)
    load, assigned, nd = (torch.empty(max(n, 1), dtype=torch.int64, device=dev) for _ in range(3))
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def maps():
        for r in range(n):
            assert L.moe_permute(p(d_ex), p(d_src), p(d_dr), i64(T), i64(E), i64(k), i64(n), i64(r), i64(n),
                                 p(rmi), p(cnt), p(oe), p(osr), p(eoff), p(nrows), p(ws), s) == 0

    def tiles():
        for r in range(n):
            assert L.moe_permute(p(d_ex), p(d_src), p(d_dr), i64(T), i64(E), i64(k), i64(n), i64(r), i64(n),
                                 p(rmi), p(cnt), p(oe), p(osr), p(eoff), p(nrows), p(ws), s) == 0
            assert L.moe_tile_layout(p(osr), p(eoff), i64(el), i64(r * el), i64(128), p(te), p(tb), p(tend),
                                     p(tm), p(nt), s) == 0

    def balance():
        assert L.moe_balance_counts(p(d_ex), p(d_dr), i64(T), i64(E), i64(k), i64(n), p(load), p(assigned),
                                    p(nd), s) == 0

    d_x = torch.from_numpy(xq).to(dev)
    nb = int(L.moe_quantize_num_blocks(i64(rows), i64(cols), 1, i64(128)))
    codes = torch.empty_like(d_x)
    scales = torch.empty(nb, dtype=torch.float64, device=dev)
    qws = torch.empty(max(int(L.moe_quantize_workspace_size(i64(rows), i64(cols), 1, i64(128))), 1),
                      dtype=torch.uint8, device=dev)

    def quant():
        assert L.moe_quantize(p(d_x), i64(rows), i64(cols), 1, i64(128), 2, p(codes), p(scales), p(qws), s) == 0

    d_v = torch.from_numpy(vec).to(dev)
    out = torch.empty(rows * cols, dtype=torch.float64, device=dev)

    def reduce():
        assert L.moe_emulate_reduce(p(d_v), i64(ranks), i64(rows * cols), 1, p(out), s) == 0

    def t(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return round(a.elapsed_time(b) / reps, 4)

    res = {"build_scatter_map_x_n_ms": t(maps), "sort_tokens_for_tiles_x_n_ms": round(t(tiles) - t(maps), 4),
           "balance_metrics_ms": t(balance), "quantize_per_token_e4m3_ms": t(quant),
           "emulate_reduce_a2a_fp32_ms": t(reduce)}
    res["total_ms"] = round(sum(v for v in res.values()), 4)
    res["note"] = ("device-resident inputs/outputs through the C ABI (binary64 numerics, bit-exact); "
                   "tiles = moe_permute + moe_tile_layout minus moe_permute")
    return res


def compare(reps_cpu=3):
    cpu, inputs = cpu_integer_path(reps=reps_cpu)
    out = {"reference_cpu": cpu}
    try:
        gpu = gpu_integer_path(inputs)
        out["ours_gpu"] = gpu
        out["speedup"] = {kk: round(cpu[kk] / gpu[kk], 1) for kk in gpu
                          if kk.endswith("_ms") and kk in cpu and gpu[kk] > 0}
    except Exception as e:  # noqa: BLE001
        out["ours_gpu"] = {"error": str(e)[:200]}
    return out


if __name__ == "__main__":
    import json
    print(json.dumps(compare()))
