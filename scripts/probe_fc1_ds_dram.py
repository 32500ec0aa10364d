"""One DeepSeek-EP4-shape fc1 grouped GEMM (64 experts x 512 rows, N 4096, K 7168,
CTA pairs) for an ncu DRAM-traffic capture (not a test). argv[1]: rows per
group list mode: 'even' (all 512) or 'odd' (alternating 384 / 640 -> M=128 tails)."""
import os
import sys
import torch
sys.path.insert(0, os.getcwd())
from paper_2505_11432_b200 import ops

G, N, K = 64, 4096, 7168
mode = sys.argv[1] if len(sys.argv) > 1 else "even"
rows_g = [512] * G if mode == "even" else [384 if g % 2 else 640 for g in range(G)]
rows = sum(rows_g)
gr = torch.tensor(rows_g, dtype=torch.int32, device="cuda")
a = torch.randn(rows, K, device="cuda").bfloat16()
b = torch.randn(G * N, K, device="cuda").bfloat16()
out = torch.empty(rows, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ops.grouped_gemm(a, b, gr, N=N, K=K, out=out, cta_pair=True)
torch.cuda.synchronize()
print("ok")
