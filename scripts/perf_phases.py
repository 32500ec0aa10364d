"""Per-phase times of the Mixtral layer (fwd+bwd), for A/B experiments (not a test)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_11432_b200.layer import MoELayer
h, f, E, k, Tr = 4096, 14336, 8, 2, 4096
g = torch.Generator(device="cuda").manual_seed(42)
w1 = (torch.randn(E, 2 * f, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
w2 = (torch.randn(E, h, f, device="cuda", generator=g) / f ** 0.5).bfloat16()
wr = (torch.randn(E, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
L = MoELayer(Tr, h, f, E, k)
L.set_weights(w1, w2, wr)
del w1, w2
x = (torch.randn(Tr, h, device="cuda", generator=g) * 0.5).bfloat16()
dy = (torch.randn(Tr, h, device="cuda", generator=g) * 0.1).bfloat16()
L.input_buffer.copy_(x)
for fused in (True, False):
    L.set_fused_dispatch(fused)
    for _ in range(3):
        L.forward(None); L.backward(dy)
    L.enable_timing(True)
    acc = {}
    for _ in range(5):
        L.forward(None); L.backward(dy)
        for kk, v in L.phase_times().items():
            acc[kk] = acc.get(kk, 0) + v / 5
    L.enable_timing(False)
    print("fused" if fused else "unfused", {kk: round(v * 1000) for kk, v in acc.items()}, "us", flush=True)
