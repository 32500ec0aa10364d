"""Warm-up + measured fwd+bwd steps of the MoE layer at EP = WORLD_SIZE (one
process per GPU, launched by torch.distributed.run) for ncu captures of the
fused kernels' NVLink traffic (never a bench number).
    argv[1] = mixtral | deepseek ; env MOE_EP_PATTERN = a2a | ag_rs"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_11432_b200.layer import MoELayer  # noqa: E402

rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
cfg = dict(h=4096, f=14336, E=8, k=2, Tr=4096)
if len(sys.argv) > 1 and sys.argv[1] == "deepseek":
    cfg = dict(h=7168, f=2048, E=256, k=8, Tr=4096)
h, f, E, k, Tr = cfg["h"], cfg["f"], cfg["E"], cfg["k"], cfg["Tr"]
el = E // n
g = torch.Generator(device="cuda").manual_seed(42)
w1 = (torch.randn(el, 2 * f, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
w2 = (torch.randn(el, h, f, device="cuda", generator=g) / f ** 0.5).bfloat16()
wr = (torch.randn(E, h, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7)) / h ** 0.5).bfloat16()
L = MoELayer(Tr, h, f, E, k, ep_size=n, rank=rank, ep_pattern=os.environ.get("MOE_EP_PATTERN", "a2a"))
L.set_weights(w1, w2, wr)
L.connect()
gx = torch.Generator(device="cuda").manual_seed(1234 + rank)
L.input_buffer.copy_((torch.randn(Tr, h, device="cuda", generator=gx) * 0.5).bfloat16())
dy = (torch.randn(Tr, h, device="cuda", generator=gx) * 0.1).bfloat16()
for _ in range(int(os.environ.get("STEPS", "2"))):
    L.forward(None)
    L.backward(dy)
L.status()
dist.barrier()
dist.destroy_process_group()
print("profile_step_ep ok", rank)
