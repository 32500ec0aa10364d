"""Grouped-GEMM throughput probe at the MoE layer's shapes (not a test)."""
import os
import sys
import torch
sys.path.insert(0, os.getcwd())
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

G, R = 8, 1024
rows = G * R
gr = torch.full((G,), R, dtype=torch.int32, device="cuda")
for name, N, K in (("fc1", 28672, 4096), ("fc2", 4096, 14336), ("sq", 8192, 8192)):
    a = torch.randn(rows, K, device="cuda").bfloat16()
    bk = torch.randn(G * N, K, device="cuda").bfloat16()
    bm = torch.randn(G * K, N, device="cuda").bfloat16()
    out = torch.empty(rows, N, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * rows * N * K
    res = {}
    for box in (0,):
        os.environ["MOE_B_BOX_ROWS"] = str(box)
        ms = timeit(lambda: ops.grouped_gemm(a, bk, gr, N=N, K=K, out=out))
        res[f"kmajor_box{box}"] = fl / ms / 1e9
    os.environ["MOE_B_BOX_ROWS"] = "0"
    ms = timeit(lambda: ops.grouped_gemm(a, bm, gr, N=N, K=K, b_mn_major=True, out=out))
    res["mnmajor"] = fl / ms / 1e9
    ms = timeit(lambda: ops.grouped_gemm(a, bk, gr, N=N, K=K, out=out, cta_pair=True))
    res["kmajor_pair"] = fl / ms / 1e9
    ms = timeit(lambda: ops.grouped_gemm(a, bm, gr, N=N, K=K, b_mn_major=True, out=out, cta_pair=True))
    res["mnmajor_pair"] = fl / ms / 1e9
    # cuBLAS reference for the same math (dense per group)
    def cub():
        for g in range(G):
            torch.matmul(a[g * R:(g + 1) * R], bk[g * N:(g + 1) * N].T, out=out[g * R:(g + 1) * R])
    ms = timeit(cub)
    res["cublas_loop"] = fl / ms / 1e9
    print(name, {k: round(v, 1) for k, v in res.items()}, "TFLOP/s", flush=True)
