"""Routing maps on the GPU, mirroring the reference's `moeplan::routing`
interface (/root/reference/proj/core/include/moeplan/routing.hpp:26-106):
same names, same argument meaning, same error behaviour (DomainError where
the reference throws std::domain_error). Every function runs the sm_100a
kernels of libmoe_b200.so; tensors live on the GPU.

Only `simulate_routing`'s RNG is not here: libstdc++ distributions are
implementation-defined, so synthetic assignments are generated on the host
(oracle/, tests) and fed in.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from ._lib import DomainError, check, i64, lib, ptr, require_cuda, stream_ptr


@dataclass
class RoutingAssignment:
    """routing.hpp:36-47 (SoA on device instead of vector<vector<int>>)."""
    num_experts: int
    top_k: int
    n_groups: int
    experts: torch.Tensor      # int32 [T, k]
    source_rank: torch.Tensor  # int32 [T]
    dropped: torch.Tensor      # uint8 [T]

    def tokens(self) -> int:
        return int(self.experts.shape[0])

    def retained_slots(self) -> int:  # routing.cpp:36-42
        return int((self.dropped == 0).sum().item()) * self.top_k

    def group_of_expert(self, expert: int) -> int:  # routing.cpp:44-47
        return expert // (self.num_experts // self.n_groups)

    @staticmethod
    def from_host(num_experts, top_k, n_groups, experts, source_rank, dropped=None, device="cuda"):
        ex = torch.as_tensor(experts, dtype=torch.int32).reshape(-1, top_k).to(device).contiguous()
        src = torch.as_tensor(source_rank, dtype=torch.int32).to(device).contiguous()
        if dropped is None:
            dr = torch.zeros(ex.shape[0], dtype=torch.uint8, device=device)
        else:
            dr = torch.as_tensor(dropped, dtype=torch.uint8).to(device).contiguous()
        return RoutingAssignment(num_experts, top_k, n_groups, ex, src, dr)


def capacity_drop(a: RoutingAssignment, capacity_factor: float, stream=None) -> torch.Tensor:
    """Group-capacity drop of routing.cpp:113-131 on the GPU; returns (and
    stores into a.dropped) the uint8 drop flags."""
    require_cuda(a.experts)
    T = a.tokens()
    dropped = torch.empty(T, dtype=torch.uint8, device=a.experts.device)
    check(lib().moe_capacity_drop(ptr(a.experts), i64(T), i64(a.num_experts), i64(a.top_k),
                                  i64(a.n_groups), __import__("ctypes").c_double(capacity_factor),
                                  ptr(dropped), stream_ptr(stream)))
    a.dropped = dropped
    return dropped


@dataclass
class ScatterMap:
    """routing.hpp:61-70."""
    my_rank: int
    rows: int
    row_map_in: torch.Tensor        # int32 [rows]  (reference: long long)
    row_map_out: torch.Tensor       # identity (routing.cpp:179)
    inverse_map: torch.Tensor       # == row_map_in (routing.cpp:180)
    per_expert_counts: torch.Tensor # int32 [E] global
    out_expert: torch.Tensor
    out_source_rank: torch.Tensor
    expert_offsets: torch.Tensor = field(default=None)  # int32 [E/n + 1]
    first_expert: int = 0


def build_scatter_map(a: RoutingAssignment, n: int, my_rank: int, stream=None) -> ScatterMap:
    """routing.hpp:72 / routing.cpp:135-187 on the GPU (bit-exact).
    Synchronises once to size the outputs, like the reference's return by
    value; the layer path never calls this (it stays on the device)."""
    require_cuda(a.experts)
    if n < 1:
        raise DomainError("n must be >= 1")
    if not (0 <= my_rank < n):
        raise DomainError("my_rank out of range")
    if a.num_experts % n != 0:
        raise DomainError("num_experts must be divisible by n")
    T, k, E = a.tokens(), a.top_k, a.num_experts
    dev = a.experts.device
    n_src = max(int(a.n_groups), int(a.source_rank.max().item()) + 1 if T else 1, 1)
    cap = max(T * k, 1)
    rmi = torch.empty(cap, dtype=torch.int32, device=dev)
    cnt = torch.empty(E, dtype=torch.int32, device=dev)
    oe = torch.empty(cap, dtype=torch.int32, device=dev)
    osr = torch.empty(cap, dtype=torch.int32, device=dev)
    offs = torch.empty(E // n + 1, dtype=torch.int32, device=dev)
    rows_d = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(int(lib().moe_permute_workspace_size(T, E, k, n_src)), dtype=torch.uint8, device=dev)
    check(lib().moe_permute(ptr(a.experts), ptr(a.source_rank), ptr(a.dropped), i64(T), i64(E),
                            i64(k), i64(n), i64(my_rank), i64(n_src), ptr(rmi), ptr(cnt), ptr(oe),
                            ptr(osr), ptr(offs), ptr(rows_d), ptr(ws), stream_ptr(stream)))
    rows = int(rows_d.item())
    rmi = rmi[:rows]
    return ScatterMap(my_rank=my_rank, rows=rows, row_map_in=rmi,
                      row_map_out=torch.arange(rows, dtype=torch.int32, device=dev),
                      inverse_map=rmi, per_expert_counts=cnt, out_expert=oe[:rows],
                      out_source_rank=osr[:rows], expert_offsets=offs,
                      first_expert=my_rank * (E // n))


@dataclass
class TileLayout:
    """routing.hpp:74-84; dependent_ranks as a bitmask per tile."""
    tile_rows: int
    expert: torch.Tensor     # int32 [tiles]
    row_begin: torch.Tensor  # int32
    row_end: torch.Tensor    # int32 (exclusive)
    rank_mask: torch.Tensor  # int64 bitmask of distinct source ranks

    def __len__(self):
        return int(self.expert.shape[0])

    def dependent_ranks(self, i: int) -> list[int]:
        m = int(self.rank_mask[i].item()) & ((1 << 64) - 1)
        return [r for r in range(64) if (m >> r) & 1]


def sort_tokens_for_tiles(m: ScatterMap, a: RoutingAssignment, tile_rows: int, stream=None) -> TileLayout:
    """routing.hpp:88-89 / routing.cpp:189-217 on the GPU (bit-exact)."""
    if tile_rows < 1:
        raise DomainError("tile_rows must be >= 1")
    dev = m.out_expert.device
    el = int(m.expert_offsets.shape[0]) - 1
    cap = max(m.rows + el, 1)
    te = torch.empty(cap, dtype=torch.int32, device=dev)
    tb = torch.empty(cap, dtype=torch.int32, device=dev)
    tend = torch.empty(cap, dtype=torch.int32, device=dev)
    tm = torch.empty(cap, dtype=torch.int64, device=dev)
    nt = torch.zeros(1, dtype=torch.int32, device=dev)
    check(lib().moe_tile_layout(ptr(m.out_source_rank), ptr(m.expert_offsets), i64(el),
                                i64(m.first_expert), i64(tile_rows), ptr(te), ptr(tb), ptr(tend),
                                ptr(tm), ptr(nt), stream_ptr(stream)))
    n_t = int(nt.item())
    return TileLayout(tile_rows, te[:n_t], tb[:n_t], tend[:n_t], tm[:n_t])


@dataclass
class BalanceStats:
    """routing.hpp:91-96."""
    per_group_load: torch.Tensor
    balance_loss_value: float
    capacity: int
    drop_rate: float


def balance_metrics(a: RoutingAssignment, n: int, stream=None) -> BalanceStats:
    """routing.hpp:101 / routing.cpp:219-262: integer counts on the GPU, the
    double arithmetic on the host in the reference's order."""
    if n < 1:
        raise DomainError("n must be >= 1")
    if not (a.n_groups == n or a.num_experts % n == 0):
        raise DomainError("incompatible group count")
    dev = a.experts.device
    load = torch.zeros(n, dtype=torch.int64, device=dev)
    assigned = torch.zeros(n, dtype=torch.int64, device=dev)
    nd = torch.zeros(1, dtype=torch.int64, device=dev)
    T = a.tokens()
    check(lib().moe_balance_counts(ptr(a.experts), ptr(a.dropped), i64(T), i64(a.num_experts),
                                   i64(a.top_k), i64(n), ptr(load), ptr(assigned), ptr(nd),
                                   stream_ptr(stream)))
    L, A, ndrop = load.cpu().tolist(), assigned.cpu().tolist(), int(nd.item())
    tl, ta = sum(L), sum(A)
    loss = 0.0
    if tl > 0 and ta > 0:
        for g in range(n):
            loss += (float(L[g]) / float(tl)) * (float(A[g]) / float(ta))
        loss *= float(n)
    cap = int(math.ceil(float(T) * float(a.top_k) / float(n))) if T > 0 else 0
    return BalanceStats(load, loss, cap, float(ndrop) / float(T) if T > 0 else 0.0)


def router_topk(x: torch.Tensor, wr: torch.Tensor, k: int, want_logits=True, stream=None):
    """K1: logits = x . wr^T (bf16 in, fp32 acc), top-k (ties -> lower id),
    gates = softmax over the k selected logits."""
    require_cuda(x, wr)
    T, h = x.shape
    E = wr.shape[0]
    dev = x.device
    logits = torch.empty(T, E, dtype=torch.float32, device=dev) if want_logits else None
    ex = torch.empty(T, k, dtype=torch.int32, device=dev)
    g = torch.empty(T, k, dtype=torch.float32, device=dev)
    check(lib().moe_router_topk(ptr(x.contiguous()), ptr(wr.contiguous()), i64(T), i64(h), i64(E),
                                i64(k), ptr(logits), ptr(ex), ptr(g), stream_ptr(stream)))
    return logits, ex, g


def topk_from_logits(logits: torch.Tensor, k: int, stream=None):
    require_cuda(logits)
    T, E = logits.shape
    ex = torch.empty(T, k, dtype=torch.int32, device=logits.device)
    g = torch.empty(T, k, dtype=torch.float32, device=logits.device)
    check(lib().moe_topk_from_logits(ptr(logits.contiguous()), i64(T), i64(E), i64(k), ptr(ex),
                                     ptr(g), stream_ptr(stream)))
    return ex, g
