"""Probe (not the product): at N = 1, fused dispatch (comm warps copy the
permuted rows inside fc1 / fc2-dgrad) vs the separate dispatch kernel + plain
GEMMs, Mixtral shape, CUDA-graph replays interleaved over rounds, plus the
per-phase times of one eager step of each.
Usage: python scripts/probe_fused_n1.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2505_11432_b200.layer import MoELayer  # noqa: E402

h, f, E, k, Tr = 4096, 14336, 8, 2, 4096
g = torch.Generator(device="cuda").manual_seed(42)
w1 = (torch.randn(E, 2 * f, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
w2 = (torch.randn(E, h, f, device="cuda", generator=g) / f ** 0.5).bfloat16()
wr = (torch.randn(E, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
L = MoELayer(Tr, h, f, E, k)
L.set_weights(w1, w2, wr)
x = (torch.randn(Tr, h, device="cuda", generator=g) * 0.5).bfloat16()
dy = (torch.randn(Tr, h, device="cuda", generator=g) * 0.1).bfloat16()
L.input_buffer.copy_(x)
y = torch.empty(Tr, h, dtype=torch.bfloat16, device="cuda")
dx = torch.empty_like(y)
dw1 = torch.empty_like(w1)
dw2 = torch.empty_like(w2)
dwr = torch.empty(E, h, dtype=torch.float32, device="cuda")


def step():
    L.forward(None, y)
    L.backward(dy, dx, dw1, dw2, dwr)


graphs = {}
phases = {}
for fused in (True, False):
    L.set_fused_dispatch(fused)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    L.enable_timing(True)
    step()
    phases[fused] = {kk: round(v, 4) for kk, v in L.phase_times().items()}
    L.enable_timing(False)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    graphs[fused] = gr
torch.cuda.synchronize()
res = {True: [], False: []}
for _ in range(5):
    for fused in (True, False):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        graphs[fused].replay()
        a.record()
        for _ in range(10):
            graphs[fused].replay()
        b.record()
        torch.cuda.synchronize()
        res[fused].append(round(a.elapsed_time(b) / 10, 4))
print(json.dumps({"fused_ms": res[True], "unfused_ms": res[False],
                  "phases_fused": phases[True], "phases_unfused": phases[False]}, indent=1))
