"""Multi-GPU parity of the fused Ulysses GEMM+A2A (QKV) / A2A+GEMM (out-proj)
against a plain torch fp32 reference of the same ops (one process per GPU)."""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank = int(os.environ["RANK"])
    n = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank))))
    from paper_2505_11432_b200.ulysses import UlyssesProjections
    s, h, m = 384 * n, 1024, 4            # s/n = 384 rows: one full pair tile + one M=128 tile
    nqkv = h * (m + 2) // m                 # 1536 = h (1 + 2/m); 1536/n per rank
    if nqkv % (256 * n):
        nqkv = 256 * n * ((nqkv + 256 * n - 1) // (256 * n))
    g = torch.Generator().manual_seed(0)
    x = (torch.randn(s, h, generator=g) * 0.5).bfloat16()
    wqkv = (torch.randn(nqkv, h, generator=g) / h ** 0.5).bfloat16()
    o = (torch.randn(s, h, generator=g) * 0.5).bfloat16()          # attention output, all heads
    wout = (torch.randn(h, h, generator=g) / h ** 0.5).bfloat16()
    U = UlyssesProjections(s, h, nqkv, n, rank)
    U.set_weights(wqkv.cuda(), wout.cuda())
    if n > 1:
        U.connect()
    sr, cpo, dh = s // n, nqkv // n, h // n
    xs = x[rank * sr:(rank + 1) * sr].cuda()
    oh = o[:, rank * dh:(rank + 1) * dh].contiguous().cuda()
    for _ in range(3):
        qkv = U.qkv_a2a(xs).clone()
        y = U.a2a_out_proj(oh)
    torch.cuda.synchronize()
    assert U.error_flag() == 0
    ref_qkv = (x.float() @ wqkv.float().T)[:, rank * cpo:(rank + 1) * cpo]
    ref_y = (o.float() @ wout.float().T)[rank * sr:(rank + 1) * sr]
    e1 = ((qkv.float().cpu() - ref_qkv).norm() / ref_qkv.norm()).item()
    e2 = ((y.float().cpu() - ref_y).norm() / ref_y.norm()).item()
    t = torch.tensor([e1, e2], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print("ULYSSES_RESULT", n, t.tolist(), flush=True)
        assert t[0] < 1e-2 and t[1] < 1e-2, t
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
