"""K-grouped (wgrad) GEMM throughput at the Mixtral and DeepSeek-EP4 shapes (not a test)."""
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


for name, G, R, M, N in (("mixtral fc2_wgrad", 8, 1024, 4096, 14336), ("mixtral fc1_wgrad", 8, 1024, 28672, 4096),
                         ("deepseek fc2_wgrad", 64, 512, 7168, 2048), ("deepseek fc1_wgrad", 64, 512, 4096, 7168),
                         ("deepseek fc1_wgrad R1024", 32, 1024, 4096, 7168)):
    rows = G * R
    a = torch.randn(rows, M, device="cuda").bfloat16()
    b = torch.randn(rows, N, device="cuda").bfloat16()
    gr = torch.full((G,), R, dtype=torch.int32, device="cuda")
    out = torch.empty(G * M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * rows * M * N
    ms = timeit(lambda: ops.grouped_gemm(a, b, gr, N=N, K=0, M=M, a_mn_major=True, b_mn_major=True,
                                         k_grouped=True, out=out, cta_pair=True))
    print(f"{name}: {ms:.3f} ms {fl / ms / 1e9:.0f} TFLOP/s, out {G * M * N * 2 / ms / 1e6:.0f} GB/s", flush=True)
