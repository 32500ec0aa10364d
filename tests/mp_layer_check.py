"""Multi-GPU layer parity check, one process per GPU (launched by
tests/test_gpu_multi.py through torch.distributed.run).

Every rank owns T_r tokens of a global batch and E/n experts; rank 0 gathers
y, dx, dW1, dW2 and the summed dWr and compares them with the fp32 oracle on
the whole batch (expert e's weights live on rank e // (E/n),
routing.cpp:44-47; token t belongs to rank t // T_r, routing.cpp:81).
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def main():
    rank = int(os.environ["RANK"])
    n = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2505_11432_b200.layer import MoELayer

    Tr, h, f = int(os.environ.get("MP_TR", 256)), 512, 512
    E, k = int(os.environ.get("MP_E", 8)), int(os.environ.get("MP_K", 2))
    cf = float(os.environ.get("MP_CF", "0"))
    T = Tr * n
    el = E // n
    g = torch.Generator().manual_seed(0)
    x = (torch.randn(T, h, generator=g) * 0.5).bfloat16()
    w1 = (torch.randn(E, 2 * f, h, generator=g) / h ** 0.5).bfloat16()
    w2 = (torch.randn(E, h, f, generator=g) / f ** 0.5).bfloat16()
    wr = (torch.randn(E, h, generator=g) / h ** 0.5).bfloat16()
    dy = (torch.randn(T, h, generator=g) * 0.1).bfloat16()

    gate_order = os.environ.get("MP_GATE", "before_fc2_in")
    comm = os.environ.get("MP_COMM", "bf16")
    tol = 5e-2 if comm == "fp8" else 1e-2
    L = MoELayer(Tr, h, f, E, k, ep_size=n, rank=rank, capacity_factor=cf, gate_order=gate_order,
                 comm_format=comm, ep_pattern=os.environ.get("MP_EP", "a2a"))
    L.set_weights(w1[rank * el:(rank + 1) * el].cuda(), w2[rank * el:(rank + 1) * el].cuda(), wr.cuda())
    L.connect()
    xs = x[rank * Tr:(rank + 1) * Tr].cuda()
    dys = dy[rank * Tr:(rank + 1) * Tr].cuda()
    for it in range(3):  # several iterations exercise buffer reuse + epochs
        y = L.forward(xs)
        dx, dw1, dw2, dwr = L.backward(dys)
    torch.cuda.synchronize()
    L.status()  # MoETimeout / debug-mode protocol assertion -> raises
    r = L.routing()
    ex_all = r["experts"].cpu().numpy()
    gt_all = r["gates"].cpu().numpy()
    dr_all = r["dropped"].cpu().numpy()
    lg = r["logits"].cpu().numpy()
    dg = r["dgates"].cpu().numpy()

    def gather(t):
        out = [torch.empty_like(t) for _ in range(n)]
        dist.all_gather(out, t.contiguous())
        return torch.cat(out).cpu()

    Y = gather(y).float().numpy()
    DX = gather(dx).float().numpy()
    DW1 = gather(dw1).float().numpy()
    DW2 = gather(dw2).float().numpy()
    LG = gather(torch.from_numpy(lg).cuda()).numpy()
    DG = gather(torch.from_numpy(dg).cuda()).numpy()
    dist.all_reduce(dwr)
    DWR = dwr.cpu().numpy()
    # every rank holds the same global routing table
    tab = torch.from_numpy(ex_all).cuda()
    tabs = [torch.empty_like(tab) for _ in range(n)]
    dist.all_gather(tabs, tab)
    ok = all((t.cpu().numpy() == ex_all).all() for t in tabs)
    if rank == 0:
        import pyoracle as P
        assert ok, "ranks disagree on the global routing table"
        xf, w1f, w2f, wrf = (t.float().numpy() for t in (x, w1, w2, wr))
        ga = gate_order.startswith("after")
        oy = P.orc_moe_forward(xf, ex_all, gt_all, dr_all, w1f, w2f, gate_after=ga)
        ob = P.orc_moe_backward(xf, dy.float().numpy(), ex_all, gt_all, LG, dr_all, w1f, w2f, wrf,
                                gate_after=ga)
        errs = dict(y=rel(Y, oy), dx=rel(DX, ob["dx"]), dw1=rel(DW1, ob["dw1"]), dw2=rel(DW2, ob["dw2"]),
                    dwr=rel(DWR, ob["dwr"]), dgates=rel(DG, ob["dgates"]))
        # routing maps bit-exact for every rank against the oracle
        src = (np.arange(T) // Tr).astype(np.int32)
        if cf > 0:
            assert (P.orc_capacity_drop(ex_all, E, n, cf) == dr_all).all()
        print("MP_RESULT", n, {kk: f"{v:.2e}" for kk, v in errs.items()}, "dropped", int(dr_all.sum()), flush=True)
        bad = {kk: v for kk, v in errs.items() if not v < tol}
        assert not bad, bad
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
