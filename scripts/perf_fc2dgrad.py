"""Isolates the Mixtral fc2-dgrad GEMM cost (not a test): standalone MN-major
grouped GEMM at its shape vs the layer's fused phase (dispatch + SwiGLU-bwd
epilogue), eager phase timing."""
import os
import sys
import torch
sys.path.insert(0, os.getcwd())
from paper_2505_11432_b200 import ops
from paper_2505_11432_b200.layer import MoELayer


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


G, R, N, K = 8, 1024, 14336, 4096
rows = G * R
gr = torch.full((G,), R, dtype=torch.int32, device="cuda")
a = torch.randn(rows, K, device="cuda").bfloat16()
bm = torch.randn(G * K, N, device="cuda").bfloat16()
out = torch.empty(rows, N, device="cuda", dtype=torch.bfloat16)
fl = 2.0 * rows * N * K
ms = timeit(lambda: ops.grouped_gemm(a, bm, gr, N=N, K=K, b_mn_major=True, out=out, cta_pair=True))
print(f"standalone mnmajor pair STORE_BF16: {ms:.3f} ms {fl / ms / 1e9:.0f} TFLOP/s")

h, f, E, k, Tr = 4096, 14336, 8, 2, 4096
w1 = (torch.randn(E, 2 * f, h, device="cuda") / h ** 0.5).bfloat16()
w2 = (torch.randn(E, h, f, device="cuda") / f ** 0.5).bfloat16()
wr = (torch.randn(E, h, device="cuda") / h ** 0.5).bfloat16()
L = MoELayer(Tr, h, f, E, k)
L.set_weights(w1, w2, wr)
L.input_buffer.copy_((torch.randn(Tr, h, device="cuda") * 0.5).bfloat16())
dy = (torch.randn(Tr, h, device="cuda") * 0.1).bfloat16()
for fused in (True, False):
    L.set_fused_dispatch(fused)
    L.enable_timing(True)
    ph = []
    for _ in range(4):
        L.forward(None)
        L.backward(dy)
        torch.cuda.synchronize()
        ph.append(L.phase_times())
    L.enable_timing(False)
    keys = ("fc1", "fc2", "fc2_dgrad", "fc1_dgrad", "fc2_wgrad", "fc1_wgrad")
    print("fused" if fused else "unfused", {q: round(min(p[q] for p in ph[1:]), 4) for q in keys})
