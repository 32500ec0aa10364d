"""configs[0] fp32 forward once (warm) + once measured, for ncu launch lists
(never a bench number)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
from paper_2505_11432_b200 import ops  # noqa: E402

T, h, f, E, k = 4096, 1024, 2816, 8, 2
r = np.random.default_rng(1234)
x = (r.standard_normal((T, h)) * 0.5).astype(np.float32)
w1 = (r.standard_normal((E, 2 * f, h)) / np.sqrt(h)).astype(np.float32)
w2 = (r.standard_normal((E, h, f)) / np.sqrt(f)).astype(np.float32)
wr = (r.standard_normal((E, h)) / np.sqrt(h)).astype(np.float32)
args = [torch.from_numpy(a).cuda() for a in (x, w1, w2, wr)]
for _ in range(2):
    y, ex, g, lg, dr = ops.ffn_forward_f32(*args, k)
torch.cuda.synchronize()
if len(sys.argv) > 1 and sys.argv[1] == "err":
    import pyoracle as P
    s = np.arange(0, T, 7)
    oy = P.orc_moe_forward(x, ex.cpu().numpy(), g.cpu().numpy(), dr.cpu().numpy(), w1, w2, tokens=s)
    print("ERR", np.linalg.norm(y.cpu().numpy()[s] - oy) / np.linalg.norm(oy))
print("probe_f32 ok")
