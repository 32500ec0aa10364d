"""Per-kernel timing of the memory-bound layer operators (not a test)."""
import os, sys, ctypes as C
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_11432_b200 import routing as R
from paper_2505_11432_b200.layer import MoELayer
T, h, E, k = 4096, 4096, 8, 2
x = (torch.randn(T, h, device="cuda") * 0.5).bfloat16()
wr = (torch.randn(E, h, device="cuda") / h ** 0.5).bfloat16()
L = MoELayer(T, h, 14336, E, k)
w1 = torch.zeros(E, 2 * 14336, h, dtype=torch.bfloat16, device="cuda"); w2 = torch.zeros(E, h, 14336, dtype=torch.bfloat16, device="cuda")
L.set_weights(w1, w2, wr); del w1, w2
L.input_buffer.copy_(x)
L.enable_timing(True)
for _ in range(5):
    L.forward(None)
print({k_: round(v * 1000, 1) for k_, v in L.phase_times().items()}, "us")
