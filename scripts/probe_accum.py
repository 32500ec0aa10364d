"""Accumulation precision of the tcgen05 bf16 GEMM: relative error against a
binary64 reference for growing K, random-sign and all-positive data."""
import numpy as np
import torch
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_11432_b200 import ops

for pos in (False, True):
    for K in (1024, 4096, 16384):
        torch.manual_seed(0)
        a = torch.randn(256, K, device="cuda")
        b = torch.randn(256, K, device="cuda")
        if pos:
            a, b = a.abs(), b.abs()
        a, b = a.bfloat16(), b.bfloat16()
        gr = torch.tensor([256], dtype=torch.int32, device="cuda")
        for cg in (False, True):
            out = ops.grouped_gemm(a, b, gr, N=256, K=K, out_dtype=torch.float32, cta_pair=cg)
            ref = a.double().cpu() @ b.double().cpu().T
            d = (out.double().cpu() - ref)
            print(f"pos={pos} K={K} cta_pair={cg} rel_l2={(d.norm() / ref.norm()).item():.3e} "
                  f"mean_signed_rel={(d / ref.abs().clamp_min(1e-30)).mean().item():.3e}")
