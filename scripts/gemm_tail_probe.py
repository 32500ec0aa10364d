"""Probe (not the product): cost of a group's M = 128 tail block in the
grouped GEMM, and the short-K / wide-N shapes (fc1, fc2 dgrad) against
torch._grouped_mm on the same box. Rows per expert 1024 (no tail), 1152
(4 pair tiles + one M = 128 pair tile), 1280 (5 pair tiles); measurements
interleaved over rounds so clock drift hits every variant alike.
Usage: python scripts/gemm_tail_probe.py [--ncu]   (--ncu: one launch each, for ncu)"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_11432_b200 import ops  # noqa: E402


def bench(fn, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ncu = "--ncu" in sys.argv
    h, f, G = 4096, 14336, 8
    g = torch.Generator(device="cuda").manual_seed(0)

    def rnd(*s):
        return (torch.randn(*s, device="cuda", generator=g) * 0.1).bfloat16()

    w1 = rnd(G, 2 * f, h)
    w2 = rnd(G, h, f)
    w1f, w2f = w1.reshape(G * 2 * f, h), w2.reshape(G * h, f)
    w1t = w1.transpose(1, 2)
    cases = {}
    for rows in (1024, 1152, 1280):
        x = rnd(rows * G, h)
        grows = torch.full((G,), rows, device="cuda", dtype=torch.int32)
        offs = grows.cumsum(0).to(torch.int32)
        o1 = torch.empty(rows * G, 2 * f, device="cuda", dtype=torch.bfloat16)
        o2 = torch.empty(rows * G, f, device="cuda", dtype=torch.bfloat16)
        cases[f"fc1_r{rows}_ours"] = (lambda x=x, gr=grows, o=o1: ops.grouped_gemm(
            x, w1f, gr, N=2 * f, K=h, cta_pair=True, out=o), 2.0 * rows * G * h * 2 * f)
        cases[f"fc1_r{rows}_torch"] = (lambda x=x, of=offs: torch._grouped_mm(x, w1t, offs=of),
                                       2.0 * rows * G * h * 2 * f)
        cases[f"fc2dg_r{rows}_ours"] = (lambda x=x, gr=grows, o=o2: ops.grouped_gemm(
            x, w2f, gr, N=f, K=h, b_mn_major=True, cta_pair=True, out=o), 2.0 * rows * G * h * f)
        cases[f"fc2dg_r{rows}_torch"] = (lambda x=x, of=offs: torch._grouped_mm(x, w2, offs=of),
                                         2.0 * rows * G * h * f)
    if ncu:
        for name, (fn, _) in cases.items():
            fn()
        torch.cuda.synchronize()
        return
    for name, (fn, _) in cases.items():
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    res = {k: [] for k in cases}
    for _ in range(4):
        for name, (fn, fl) in cases.items():
            ms = bench(fn, 10)
            res[name].append(round(fl / ms / 1e9, 1))
    out = {k: {"tflops_rounds": v, "median": sorted(v)[len(v) // 2]} for k, v in res.items()}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
