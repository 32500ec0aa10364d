"""Comparison baseline (NOT the product): the six expert GEMMs of one MoE
layer step (fc1, fc2, fc2 dgrad, fc1 dgrad, fc2 wgrad, fc1 wgrad;
graph.cpp:288-296, 376-398) at identical bf16 shapes through
  - torch._grouped_mm (CUTLASS grouped GEMM shipped with torch),
  - per-expert cuBLAS (torch.matmul on each expert's rows),
  - this repo's tcgen05 grouped GEMM as a plain GEMM (moe_grouped_gemm, no
    fused dispatch / SwiGLU / scatter epilogues; expert segments padded to 128
    rows as the layer runs them).
Used by bench.py (`gemm_vs_cublas`) on the same box and data; times are CUDA
events over `reps` back-to-back launches after warm-up, inputs > L2.
"""
from __future__ import annotations

import torch


def _time(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def compare_gemms(h: int, f: int, counts: list[int], reps: int = 10, seed: int = 0):
    from paper_2505_11432_b200 import ops
    dev = "cuda"
    G = len(counts)
    rows = sum(counts)
    pad = [(c + 127) // 128 * 128 for c in counts]
    prow = sum(pad)
    g = torch.Generator(device=dev).manual_seed(seed)

    def rnd(*s):
        return (torch.randn(*s, device=dev, generator=g) * 0.1).bfloat16()

    w1 = rnd(G, 2 * f, h)
    w2 = rnd(G, h, f)
    x, dy = rnd(rows, h), rnd(rows, h)
    z, dh = rnd(rows, f), rnd(rows, 2 * f)
    xp, dyp, zp, dhp = rnd(prow, h), rnd(prow, h), rnd(prow, f), rnd(prow, 2 * f)
    offs = torch.tensor(counts, device=dev, dtype=torch.int32).cumsum(0).to(torch.int32)
    grows = torch.tensor(pad, device=dev, dtype=torch.int32)
    starts = [0]
    for c in counts:
        starts.append(starts[-1] + c)
    flops = {
        "fc1": 2.0 * rows * h * 2 * f, "fc2": 2.0 * rows * f * h, "fc2_dgrad": 2.0 * rows * h * f,
        "fc1_dgrad": 2.0 * rows * 2 * f * h, "fc2_wgrad": 2.0 * rows * h * f, "fc1_wgrad": 2.0 * rows * 2 * f * h,
    }
    w1t, w2t = w1.transpose(1, 2), w2.transpose(1, 2)   # [G, h, 2f], [G, f, h]

    gm = {
        "fc1": lambda: torch._grouped_mm(x, w1t, offs=offs),
        "fc2": lambda: torch._grouped_mm(z, w2t, offs=offs),
        "fc2_dgrad": lambda: torch._grouped_mm(dy, w2, offs=offs),
        "fc1_dgrad": lambda: torch._grouped_mm(dh, w1, offs=offs),
        "fc2_wgrad": lambda: torch._grouped_mm(dy.t(), z, offs=offs),
        "fc1_wgrad": lambda: torch._grouped_mm(dh.t(), x, offs=offs),
    }

    def loop(fn):
        def run():
            for e in range(G):
                fn(e, slice(starts[e], starts[e + 1]))
        return run

    cb = {
        "fc1": loop(lambda e, s: torch.matmul(x[s], w1[e].t())),
        "fc2": loop(lambda e, s: torch.matmul(z[s], w2[e].t())),
        "fc2_dgrad": loop(lambda e, s: torch.matmul(dy[s], w2[e])),
        "fc1_dgrad": loop(lambda e, s: torch.matmul(dh[s], w1[e])),
        "fc2_wgrad": loop(lambda e, s: torch.matmul(dy[s].t(), z[s])),
        "fc1_wgrad": loop(lambda e, s: torch.matmul(dh[s].t(), x[s])),
    }
    w1f, w2f = w1.reshape(G * 2 * f, h), w2.reshape(G * h, f)
    ours = {
        "fc1": lambda: ops.grouped_gemm(xp, w1f, grows, N=2 * f, K=h, cta_pair=True),
        "fc2": lambda: ops.grouped_gemm(zp, w2f, grows, N=h, K=f, cta_pair=True),
        "fc2_dgrad": lambda: ops.grouped_gemm(dyp, w2f, grows, N=f, K=h, b_mn_major=True, cta_pair=True),
        "fc1_dgrad": lambda: ops.grouped_gemm(dhp, w1f, grows, N=h, K=2 * f, b_mn_major=True, cta_pair=True),
        "fc2_wgrad": lambda: ops.grouped_gemm(dyp, zp, grows, M=h, N=f, K=0, a_mn_major=True, b_mn_major=True,
                                              k_grouped=True, cta_pair=True),
        "fc1_wgrad": lambda: ops.grouped_gemm(dhp, xp, grows, M=2 * f, N=h, K=0, a_mn_major=True, b_mn_major=True,
                                              k_grouped=True, cta_pair=True),
    }
    out = {}
    for name in flops:
        res = {}
        for impl, table in (("ours_plain", ours), ("torch_grouped_mm", gm), ("cublas_per_expert", cb)):
            try:
                ms = _time(table[name], reps)
                res[impl] = {"ms": round(ms, 4), "tflops": round(flops[name] / ms / 1e9, 1)}
            except Exception as ex:  # noqa: BLE001
                res[impl] = {"error": str(ex).splitlines()[0][:160]}
        out[name] = res
    tot = {impl: sum(out[nm][impl].get("ms", float("nan")) for nm in flops)
           for impl in ("ours_plain", "torch_grouped_mm", "cublas_per_expert")}
    return {"shapes": {"h": h, "f": f, "experts": G, "rows_per_expert": counts},
            "per_gemm": out, "sum_ms": {k: round(v, 4) for k, v in tot.items()},
            "note": "same bf16 shapes on the same box; ours_plain = moe_grouped_gemm without the layer's fused "
                    "epilogues (rows padded to 128 per expert); the layer's fused GEMMs are in phases_ms"}


if __name__ == "__main__":
    import json
    print(json.dumps(compare_gemms(4096, 14336, [1024] * 8)))
