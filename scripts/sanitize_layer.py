"""Small MoE layer fwd+bwd (bf16 and FP8 comm, CTA-pair and single-CTA tiles,
fused dispatch with dedup at EP > 1) for compute-sanitizer runs
(scripts/sanitize.sh). Under torch.distributed.run it runs at EP = WORLD_SIZE."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_11432_b200.layer import MoELayer  # noqa: E402

n = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
if n > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))))
cases = [dict(T=256, h=512, f=512, E=8, k=2, comm="bf16", gate="before_fc2_in"),
         dict(T=512, h=512, f=256, E=16, k=4, comm="bf16", gate="before_fc2_in"),
         dict(T=256, h=512, f=512, E=8, k=2, comm="fp8", gate="after_fc2_out")]
for c in cases:
    g = torch.Generator(device="cuda").manual_seed(1)
    el = c["E"] // n
    L = MoELayer(c["T"], c["h"], c["f"], c["E"], c["k"], ep_size=n, rank=rank, capacity_factor=1.25,
                 comm_format=c["comm"], gate_order=c["gate"])
    L.set_weights((torch.randn(el, 2 * c["f"], c["h"], device="cuda", generator=g) * 0.05).bfloat16(),
                  (torch.randn(el, c["h"], c["f"], device="cuda", generator=g) * 0.05).bfloat16(),
                  (torch.randn(c["E"], c["h"], device="cuda", generator=g) * 0.05).bfloat16())
    if n > 1:
        L.connect()
    x = (torch.randn(c["T"], c["h"], device="cuda", generator=g) * 0.5).bfloat16()
    dy = (torch.randn(c["T"], c["h"], device="cuda", generator=g) * 0.1).bfloat16()
    for _ in range(2):
        L.forward(x)
        L.backward(dy)
    L.status()
    del L
    torch.cuda.synchronize()
print("sanitize_layer ok", rank, flush=True)
if n > 1:
    dist.barrier()
    dist.destroy_process_group()
