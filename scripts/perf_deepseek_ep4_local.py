"""Per-phase times of one rank's DeepSeek EP=4 expert work (64 experts, k=8) on one GPU (not a test)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2505_11432_b200.layer import MoELayer
h, f, E, k, Tr = 7168, 2048, 64, 8, 4096
g = torch.Generator(device="cuda").manual_seed(42)
w1 = (torch.randn(E, 2 * f, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
w2 = (torch.randn(E, h, f, device="cuda", generator=g) / f ** 0.5).bfloat16()
wr = (torch.randn(E, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
L = MoELayer(Tr, h, f, E, k); L.set_weights(w1, w2, wr)
L.input_buffer.copy_((torch.randn(Tr, h, device="cuda") * 0.5).bfloat16())
dy = (torch.randn(Tr, h, device="cuda") * 0.1).bfloat16()
L.enable_timing(True)
ph=[]
for _ in range(4):
    L.forward(None); L.backward(dy); torch.cuda.synchronize(); ph.append(L.phase_times())
print({q: round(min(p[q] for p in ph[1:]), 4) for q in ph[0]})
