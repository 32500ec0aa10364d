"""Multi-GPU parity of the fused attention AG-GEMM / GEMM-RS against a plain
torch fp32 reference of the same ops (one process per GPU)."""
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
    from paper_2505_11432_b200.attn import AttnProjections
    s, h = int(os.environ.get("MP_ATTN_S", 1024 * n)), 1024
    nq = int(os.environ.get("MP_ATTN_NQ", 256 * 5 // 2 if n == 1 else 320))  # any multiple of 64
    g = torch.Generator().manual_seed(0)
    x = (torch.randn(s, h, generator=g) * 0.5).bfloat16()
    wqkv = (torch.randn(n, nq, h, generator=g) / h ** 0.5).bfloat16()
    o = (torch.randn(s, h, generator=g) * 0.5).bfloat16()          # attention output, all heads
    wout = (torch.randn(h, h, generator=g) / h ** 0.5).bfloat16()   # [out, in]
    A = AttnProjections(s, h, nq, n, rank)
    dh = h // n
    A.set_weights(wqkv[rank].cuda(), wout[:, rank * dh:(rank + 1) * dh].contiguous().cuda())
    if n > 1:
        A.connect()
    sr = s // n
    for _ in range(3):
        qkv = A.ag_gemm(x[rank * sr:(rank + 1) * sr].cuda())
        y = A.gemm_rs(o[:, rank * dh:(rank + 1) * dh].contiguous().cuda())
    torch.cuda.synchronize()
    assert A.error_flag() == 0
    # the fused GEMM-RS (reduction in the own-shard tiles' epilogue) against the
    # unfused staging + barrier + reduce kernel: same partials, same rank order
    os.environ["MOE_ATTN_RS_UNFUSED"] = "1"
    B = AttnProjections(s, h, nq, n, rank)
    del os.environ["MOE_ATTN_RS_UNFUSED"]
    B.set_weights(wqkv[rank].cuda(), wout[:, rank * dh:(rank + 1) * dh].contiguous().cuda())
    if n > 1:
        B.connect()
    y_unfused = B.gemm_rs(o[:, rank * dh:(rank + 1) * dh].contiguous().cuda())
    torch.cuda.synchronize()
    assert B.error_flag() == 0
    same = torch.tensor([float(torch.equal(y, y_unfused))], device="cuda")
    dist.all_reduce(same, op=dist.ReduceOp.MIN)
    assert same.item() == 1.0, "fused GEMM-RS differs from staging + reduce"
    A.status()
    ref_qkv = x.float() @ wqkv[rank].float().T
    ref_y = (o.float() @ wout.float().T)[rank * sr:(rank + 1) * sr]
    e1 = ((qkv.float().cpu() - ref_qkv).norm() / ref_qkv.norm()).item()
    e2 = ((y.float().cpu() - ref_y).norm() / ref_y.norm()).item()
    t = torch.tensor([e1, e2], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print("ATTN_RESULT", n, t.tolist(), flush=True)
        assert t[0] < 1e-2 and t[1] < 1e-2, t
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
