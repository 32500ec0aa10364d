"""Probe (not the product): DRAM reads of the fc1-dgrad-shaped grouped GEMM
(N = 4096, K = 28672, Mixtral experts) under variations, one launch each for
ncu: argv[1] = mn8 (8 experts x 1024 rows, B MN-major as in the layer) |
km8 (B K-major copy) | mn1 (one expert, 8192 rows) | mn8s (rows 1152, tails)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_11432_b200 import ops  # noqa: E402

h, f = 4096, 14336
v = sys.argv[1]
G = 1 if v == "mn1" else 8
rows = 8192 if v == "mn1" else (1152 if v == "mn8s" else 1024)
g = torch.Generator(device="cuda").manual_seed(0)
w1 = (torch.randn(G, 2 * f, h, device="cuda", generator=g) * 0.02).bfloat16()
a = (torch.randn(G * rows, 2 * f, device="cuda", generator=g) * 0.1).bfloat16()
gr = torch.full((G,), rows, device="cuda", dtype=torch.int32)
out = torch.empty(G * rows, h, device="cuda", dtype=torch.bfloat16)
if v == "km8":
    w1t = w1.transpose(1, 2).contiguous().reshape(G * h, 2 * f)   # [G*h, 2f] K-major
    fn = lambda: ops.grouped_gemm(a, w1t, gr, N=h, K=2 * f, cta_pair=True, out=out)
else:
    w1f = w1.reshape(G * 2 * f, h)
    fn = lambda: ops.grouped_gemm(a, w1f, gr, N=h, K=2 * f, b_mn_major=True, cta_pair=True, out=out)
for _ in range(2):
    fn()
torch.cuda.synchronize()
print("ok", v)
