"""Grouped GEMM throughput at the DeepSeek-V3 per-rank shapes of EP=8
(32 local experts x ~1024 rows, h 7168, f 2048) -- not a test."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_11432_b200 import ops

def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for G, R in ((32, 1024), (64, 512), (8, 1024)):
    rows = G * R
    gr = torch.full((G,), R, dtype=torch.int32, device="cuda")
    for name, N, K in (("fc1", 4096, 7168), ("fc2", 7168, 2048), ("fc2_dgrad(MN B)", 2048, 7168)):
        a = torch.randn(rows, K, device="cuda").bfloat16()
        bk = torch.randn(G * N, K, device="cuda").bfloat16()
        bm = torch.randn(G * K, N, device="cuda").bfloat16()
        out = torch.empty(rows, N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * rows * N * K
        res = {}
        for cp in (False, True):
            if R % (256 if cp else 128):
                continue
            if "MN" in name:
                ms = timeit(lambda: ops.grouped_gemm(a, bm, gr, N=N, K=K, b_mn_major=True, out=out, cta_pair=cp))
            else:
                ms = timeit(lambda: ops.grouped_gemm(a, bk, gr, N=N, K=K, out=out, cta_pair=cp))
            res["pair" if cp else "single"] = round(fl / ms / 1e9, 1)
        print(f"G={G} R={R} {name}", res, "TFLOP/s", flush=True)
        del a, bk, bm, out
