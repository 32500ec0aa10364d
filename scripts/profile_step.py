"""One warm-up + one measured fwd+bwd step of the Mixtral-shape layer, for
ncu launch lists / captures (never a bench number)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_11432_b200.layer import MoELayer

cfg = dict(h=4096, f=14336, E=8, k=2, Tr=4096)
if len(sys.argv) > 1 and sys.argv[1] == "deepseek":
    cfg = dict(h=7168, f=2048, E=256, k=8, Tr=4096)
if len(sys.argv) > 1 and sys.argv[1] == "deepseek_ep4":
    # one rank's expert work at EP = 4 (64 local experts, ~512 rows each) on one GPU
    cfg = dict(h=7168, f=2048, E=64, k=8, Tr=4096)
h, f, E, k, Tr = cfg["h"], cfg["f"], cfg["E"], cfg["k"], cfg["Tr"]
g = torch.Generator(device="cuda").manual_seed(42)
w1 = (torch.randn(E, 2 * f, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
w2 = (torch.randn(E, h, f, device="cuda", generator=g) / f ** 0.5).bfloat16()
wr = (torch.randn(E, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
L = MoELayer(Tr, h, f, E, k)
L.set_weights(w1, w2, wr)
x = (torch.randn(Tr, h, device="cuda", generator=g) * 0.5).bfloat16()
dy = (torch.randn(Tr, h, device="cuda", generator=g) * 0.1).bfloat16()
L.input_buffer.copy_(x)
steps = int(os.environ.get("STEPS", "2"))
for _ in range(steps):
    L.forward(None)
    L.backward(dy)
torch.cuda.synchronize()
print("profile_step ok")
