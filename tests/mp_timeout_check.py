"""MOE_ERR_TIMEOUT end to end (tests/test_gpu_multi.py): rank 1 connects and
then never calls forward; rank 0's flag barriers give up after
MOE_FLAG_TIMEOUT_MS and moe_layer_status reports MOE_ERR_TIMEOUT (Python
MoETimeout), and the next forward refuses to run until clear_error."""
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    from paper_2505_11432_b200 import MoETimeout
    from paper_2505_11432_b200.layer import MoELayer
    Tr, h, f, E, k = 256, 512, 512, 8, 2
    g = torch.Generator(device="cuda").manual_seed(0)
    L = MoELayer(Tr, h, f, E, k, ep_size=n, rank=rank)
    el = E // n
    L.set_weights((torch.randn(el, 2 * f, h, device="cuda", generator=g) * 0.05).bfloat16(),
                  (torch.randn(el, h, f, device="cuda", generator=g) * 0.05).bfloat16(),
                  (torch.randn(E, h, device="cuda", generator=g) * 0.05).bfloat16())
    L.connect()
    dist.barrier()
    if rank == 0:
        x = (torch.randn(Tr, h, device="cuda", generator=g) * 0.5).bfloat16()
        t0 = time.time()
        L.forward(x)                     # rank 1 never arrives
        try:
            L.status()
            ok = False
        except MoETimeout as e:
            ok = True
            print("TIMEOUT_RAISED", f"{time.time() - t0:.1f}s", str(e)[:120], flush=True)
        assert ok, "status() did not report the timeout"
        try:
            L.forward(x)
            refused = False
        except MoETimeout:
            refused = True
        assert refused, "forward ran on after a timeout"
        L.clear_error()
        print("TIMEOUT_RESULT ok", flush=True)
    dist.barrier()          # rank 1 keeps its buffers mapped until rank 0 is done
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
