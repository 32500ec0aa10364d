"""Full-shape sampled parity of the MoE layer with EP over NVLink, one process
per GPU (launched by tests/test_gpu_multi.py through torch.distributed.run).

Every rank owns T_r = 4096 tokens of the global batch (token t on rank
t // T_r, routing.cpp:81) and E/n experts (expert e on rank e // (E/n),
routing.cpp:44-47). Each rank checks its own scatter map bit-exact against
the oracle; rank 0 gathers y, dx, dgates, logits, the sampled wgrad columns of
every expert and the summed dW_r and compares them with the binary64 oracle
(sampling and tolerances: tests/fullshape_common.py).
  MP_CFG = cfg2_mixtral | cfg3_deepseek | cfg5_fp8_zipf
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

from fullshape_common import (CONFIGS, check_dropped_zero, check_routing, dense_errors, make_inputs,  # noqa: E402
                              sample, tolerance, wgrad_cols, zipf_routing)


def main():
    rank = int(os.environ["RANK"])
    n = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import pyoracle as P
    from paper_2505_11432_b200.layer import MoELayer
    name = os.environ.get("MP_CFG", "cfg2_mixtral")
    c = CONFIGS[name]
    Tr = int(os.environ.get("MP_TR", 4096))
    h, f, E, k = c["h"], c["f"], c["E"], c["k"]
    T, el = Tr * n, E // n
    w1, w2, wr, x, dy = make_inputs(c, T)
    L = MoELayer(Tr, h, f, E, k, ep_size=n, rank=rank, capacity_factor=c.get("cf", 0.0),
                 route_mode="injected" if c["route"] == "zipf" else "learned",
                 gate_order=c["gate"], comm_format=c["comm"], ep_pattern=os.environ.get("MP_EP", "a2a"))
    L.set_weights(w1[rank * el:(rank + 1) * el].contiguous(), w2[rank * el:(rank + 1) * el].contiguous(), wr)
    L.connect()
    if c["route"] == "zipf":
        from conftest import GOLDEN
        ex_in, gt_in = zipf_routing(GOLDEN, T, k)
        L.set_routing(torch.from_numpy(ex_in[rank * Tr:(rank + 1) * Tr]).cuda(),
                      torch.from_numpy(gt_in[rank * Tr:(rank + 1) * Tr]).cuda())
    sl = slice(rank * Tr, (rank + 1) * Tr)
    for _ in range(2):  # a second step exercises buffer reuse and epochs
        y = L.forward(x[sl].contiguous())
        dx, dw1, dw2, dwr = L.backward(dy[sl].contiguous())
    L.status()
    r = L.routing()
    ex, gt, dr = (r[q].cpu().numpy() for q in ("experts", "gates", "dropped"))
    if c.get("cf", 0.0) > 0:
        # the layer's drops (replicated on every rank) = the pinned oracle's, routing.cpp:113-131
        assert (P.orc_capacity_drop(ex, E, n, c["cf"]) == dr).all(), "capacity drops differ from the oracle"
    else:
        assert dr.sum() == 0
    toks, cols = sample(T, f, n_col=4, dropped=dr if c.get("cf", 0.0) > 0 else None)

    def gather(t):
        out = [torch.empty_like(t) for _ in range(n)]
        dist.all_gather(out, t.contiguous())
        return torch.cat(out).cpu()

    Y = gather(y).float().numpy()
    DX = gather(dx).float().numpy()
    LG = gather(r["logits"]).numpy()
    DG = gather(r["dgates"]).numpy()
    g1, g2 = wgrad_cols(dw1, dw2, cols, f)
    G1, G2 = gather(g1).numpy(), gather(g2).numpy()
    dist.all_reduce(dwr)
    # every rank: the global routing table agrees and its own scatter map is bit-exact
    tabs = gather(torch.from_numpy(ex).cuda()).numpy().reshape(n, T, k)
    assert all((t == ex).all() for t in tabs), "ranks disagree on the global routing table"
    lerr = None
    if rank == 0:
        lerr, maps = check_routing(P, c, ex, gt, dr, LG, toks, x, wr, n, Tr)
    else:
        src = (np.arange(T) // Tr).astype(np.int32)
        maps = {rank: P.orc_build_scatter_map(ex, src, dr, E, n, rank)}
    m = maps[rank]
    ok = (r["row_map_in"].cpu().numpy() == m["row_map_in"]).all() and \
         (r["per_expert_counts"].cpu().numpy() == m["per_expert_counts"]).all()
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(flag)
    assert flag.item() == 0, "a rank's scatter map differs from the oracle"
    if rank == 0:
        errs = {}
        if c.get("cf", 0.0) > 0:
            check_dropped_zero(dr, Y, DX, DG)
        if lerr is not None:
            errs["logits"] = lerr
            assert lerr < 1e-4, errs
        errs.update(dense_errors(P, c, ex, gt, dr, DG, toks, cols, x, dy, w1, w2, wr, Y[toks], DX[toks],
                                 G1, G2, dwr.cpu().numpy()))
        rows = [int((np.asarray(r2["row_map_in"]).size)) for r2 in maps]
        print("MP_FULL_RESULT", name, n, {kk: f"{v:.2e}" for kk, v in errs.items()}, "rows_per_rank", rows,
              "dropped_tokens", int(dr.sum()), flush=True)
        bad = {kk: v for kk, v in errs.items() if kk != "logits" and not v < tolerance(c, kk)}
        assert not bad, bad
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
