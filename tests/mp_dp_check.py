"""Multi-GPU parity of the compressed DP reduce-scatter / all-gather
(moe_dp_*) against the oracle's emulate_reduce(a2a_fp32) (bit-exact), one
process per GPU."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def grads_of(rank, count):
    g = np.random.default_rng(100 + rank)
    mag = 10.0 ** g.uniform(-6, 4, count)
    v = (g.standard_normal(count) * mag).astype(np.float32)
    v[:7] = [0.0, -0.0, 1e-40, -3e-39, 65504.0, 3.3e38, -1.0]   # zeros, fp32 subnormals, large
    return v


def main():
    rank = int(os.environ["RANK"])
    n = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank))))
    import pyoracle as P
    from paper_2505_11432_b200.dp import DpGradSync
    count = 4096 * n * 24
    S = count // n
    D = DpGradSync(count, n, rank)
    if n > 1:
        D.connect()
    allg = np.stack([grads_of(p, count) for p in range(n)])

    def reduced(p):
        part = allg[:, p * S:(p + 1) * S].astype(np.float64)
        if n == 1:   # one rank: the bf16 round trip (round_to is the reduction's input rounding)
            return P.orc_round_to("bf16", part[0]).astype(np.float32)
        with np.errstate(over="ignore"):
            return P.orc_emulate_reduce(part, "a2a_fp32").astype(np.float32)
    want = reduced(rank)
    ok = True
    for it in range(3):
        D.grad.copy_(torch.from_numpy(allg[rank]).cuda())
        shard = D.reduce_scatter()
        got = shard.cpu().numpy()
        eq = np.array_equal(got.view(np.uint32), want.view(np.uint32))
        if not eq:
            bad = np.nonzero(got.view(np.uint32) != want.view(np.uint32))[0]
            print(f"rank {rank} it {it}: {len(bad)} mismatches, first {bad[:5]} got {got[bad[:5]]} want {want[bad[:5]]}",
                  flush=True)
        ok &= bool(eq)
        upd = (shard * 0.5).contiguous()
        full = D.all_gather_bf16(upd)
        exp_full = torch.cat([torch.from_numpy(reduced(p)) * 0.5 for p in range(n)]).bfloat16()
        eqf = torch.equal(full.cpu().view(torch.int16), exp_full.view(torch.int16))
        if not eqf:
            bad = torch.nonzero(full.cpu().view(torch.int16) != exp_full.view(torch.int16)).flatten()
            print(f"rank {rank} it {it}: all-gather {bad.numel()} mismatches, first {bad[:5].tolist()}", flush=True)
        ok &= bool(eqf)
    torch.cuda.synchronize()
    ok &= D.error_flag() == 0
    t = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(t)
    if rank == 0:
        print("DP_RESULT", n, int(t.item()), flush=True)
        assert t.item() == 0
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
