"""MoE layer (reference operator chain ffn_norm? -> router -> dispatch ->
fc1 -> swiglu -> weighted_sum -> fc2 -> gather/combine, graph.cpp:254-311,
and its backward, graph.cpp:333-401) as a handle over the C ABI.

Multi-GPU: one process per GPU; `MoELayer.connect(group)` exchanges the
CUDA-IPC handles of every rank's symmetric arena over torch.distributed, after
which dispatch/combine run as in-kernel NVLink loads/stores.
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import DomainError, check, i64, lib, ptr, require_cuda, stream_ptr


class _Cfg(C.Structure):
    _fields_ = [("tokens_per_rank", C.c_int64), ("hidden", C.c_int64), ("ffn_hidden", C.c_int64),
                ("num_experts", C.c_int64), ("top_k", C.c_int64), ("ep_size", C.c_int64),
                ("rank", C.c_int64), ("capacity_factor", C.c_double), ("gate_order", C.c_int32),
                ("comm_format", C.c_int32), ("ep_pattern", C.c_int32), ("route_mode", C.c_int32),
                ("ffn_norm", C.c_int32), ("norm_eps", C.c_float), ("no_remat", C.c_int32)]


class _RoutingView(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("experts", "gates", "dropped", "row_map_in",
                                          "per_expert_counts", "out_expert", "out_source_rank",
                                          "rows", "dgates", "logits")]


class _DevArray:
    """Zero-copy view of layer-owned device memory (CUDA array interface)."""

    def __init__(self, p, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(p), False), "version": 3, "strides": None}


def _view(p, shape, dtype):
    typestr = {torch.int32: "<i4", torch.float32: "<f4", torch.uint8: "|u1",
               torch.bfloat16: "<u2"}[dtype]
    t = torch.as_tensor(_DevArray(p, shape, typestr), device="cuda")
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


def _check(t, shape, dtype, name):
    """Shape / dtype / layout of a tensor handed to the C ABI as a raw pointer."""
    if t is None:
        return None
    require_cuda(t)
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype:
        raise DomainError(f"{name} must be {dtype} {list(shape)}, got {t.dtype} {list(t.shape)}")
    if not t.is_contiguous():
        raise DomainError(f"{name} must be contiguous")
    return t


EP_PATTERNS = {"a2a": 0, "ag_rs": 1}   # commcost.hpp:81 EpPattern order
GATE_ORDERS = {"before_fc2_in": 0, "before_fc2": 0, "after_fc2_out": 1, "after_fc2": 1}


class MoELayer:
    def __init__(self, tokens_per_rank: int, hidden: int, ffn_hidden: int, num_experts: int,
                 top_k: int, ep_size: int = 1, rank: int = 0, capacity_factor: float = 0.0,
                 gate_order: str = "before_fc2_in", comm_format: str = "bf16",
                 route_mode: str = "learned", ffn_norm: bool = False, norm_eps: float = 1e-6,
                 ep_pattern: str = "a2a", remat: bool = True):
        """ep_pattern (commcost.hpp:81): "a2a" = pull only the rows this rank's
        experts need + push every (token, slot) output row to its owner;
        "ag_rs" = all-gather every token row, local scatter, and one
        pre-reduced partial row per (token, serving rank) reduce-scattered to
        the owner (bf16 communication, gate before fc2).
        remat (memmodel.cpp:25-31, main.cpp `--no-remat`): True = selective
        rematerialisation, fc2_in recomputed in backward (the reference
        default); False = the forward's fc2_in is kept and reused."""
        cfg = _Cfg(tokens_per_rank, hidden, ffn_hidden, num_experts, top_k, ep_size, rank,
                   float(capacity_factor), GATE_ORDERS[gate_order],
                   {"bf16": 0, "fp8": 1, "fp8_e4m3": 1}[comm_format], EP_PATTERNS[ep_pattern],
                   {"learned": 0, "injected": 1}[route_mode], int(bool(ffn_norm)), float(norm_eps),
                   int(not remat))
        self.norm = bool(ffn_norm)
        self.cfg = cfg
        self.Tr, self.h, self.f, self.E, self.k = tokens_per_rank, hidden, ffn_hidden, num_experts, top_k
        self.n, self.rank = ep_size, rank
        self.el = num_experts // ep_size
        h_ = C.c_void_p()
        check(lib().moe_layer_create(C.byref(cfg), C.byref(h_)))
        self._h = h_
        self._x_in = _view(lib().moe_layer_input_buffer(self._h), (tokens_per_rank, hidden), torch.bfloat16)
        # symmetric dy buffer: writing dy here and passing it to backward skips a copy
        self.dy_buffer = _view(lib().moe_layer_dy_buffer(self._h), (tokens_per_rank, hidden), torch.bfloat16)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().moe_layer_destroy(h)
            self._h = None

    # ------------------------------------------------------------------
    @property
    def input_buffer(self) -> torch.Tensor:
        """[T_r, h] bf16 view of the layer's symmetric input buffer."""
        return self._x_in

    def set_weights(self, w1: torch.Tensor, w2: torch.Tensor, wr: torch.Tensor | None = None, stream=None):
        """w1 [E_local, 2f, h] ([a | b] rows), w2 [E_local, h, f], wr [E, h]; bf16."""
        require_cuda(w1, w2, wr)
        if w1.dtype != torch.bfloat16 or w2.dtype != torch.bfloat16 or (wr is not None and wr.dtype != torch.bfloat16):
            raise DomainError("weights must be bf16")
        if w1.shape != (self.el, 2 * self.f, self.h) or w2.shape != (self.el, self.h, self.f):
            raise DomainError("weight shapes must be w1 [E/n, 2f, h], w2 [E/n, h, f]")
        if wr is not None and wr.shape != (self.E, self.h):
            raise DomainError("router weight must be [E, h]")
        self._keep = (w1.contiguous(), w2.contiguous(), None if wr is None else wr.contiguous())
        check(lib().moe_layer_set_weights(self._h, ptr(self._keep[0]), ptr(self._keep[1]),
                                          ptr(self._keep[2]), stream_ptr(stream)))

    def set_norm_weight(self, gamma: torch.Tensor, stream=None):
        """ffn_norm weight [h] (fp32)."""
        require_cuda(gamma)
        self._gamma = gamma.float().contiguous()
        check(lib().moe_layer_set_norm_weight(self._h, ptr(self._gamma), stream_ptr(stream)))

    def norm_grad(self) -> torch.Tensor:
        lib().moe_layer_norm_grad.restype = C.c_void_p
        return _view(lib().moe_layer_norm_grad(self._h), (self.h,), torch.float32)

    def set_routing(self, experts: torch.Tensor, gates: torch.Tensor, stream=None):
        require_cuda(experts, gates)
        if tuple(experts.shape) != (self.Tr, self.k) or tuple(gates.shape) != (self.Tr, self.k):
            raise DomainError(f"experts / gates must be [{self.Tr}, {self.k}]")
        self._route_keep = (experts.to(torch.int32).contiguous(), gates.float().contiguous())
        check(lib().moe_layer_set_routing(self._h, ptr(self._route_keep[0]), ptr(self._route_keep[1]),
                                          stream_ptr(stream)))

    def forward(self, x: torch.Tensor | None, y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        if x is not None:
            require_cuda(x)
            x = _check(x.contiguous(), (self.Tr, self.h), torch.bfloat16, "x")
        if y is None:
            y = torch.empty(self.Tr, self.h, dtype=torch.bfloat16, device="cuda")
        _check(y, (self.Tr, self.h), torch.bfloat16, "y")
        check(lib().moe_layer_forward(self._h, ptr(x), ptr(y), stream_ptr(stream)))
        return y

    # the forward as the reference's fused pairs (moe_layer_route / moe_dispatch_fc1 /
    # moe_fc2_combine; schedule.cpp:205-272)
    def route(self, x: torch.Tensor | None, stream=None):
        """K1+K2: router, routing metadata, capacity drop, permutation."""
        if x is not None:
            x = _check(x.contiguous(), (self.Tr, self.h), torch.bfloat16, "x")
        check(lib().moe_layer_route(self._h, ptr(x), stream_ptr(stream)))

    def dispatch_fc1(self, stream=None):
        """K3: AG + local scatter fused into fc1 + SwiGLU (+ gate)."""
        check(lib().moe_dispatch_fc1(self._h, stream_ptr(stream)))

    def fc2_combine(self, y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """K4+K5: fc2 with the gather / RS epilogue, then the combine."""
        if y is None:
            y = torch.empty(self.Tr, self.h, dtype=torch.bfloat16, device="cuda")
        _check(y, (self.Tr, self.h), torch.bfloat16, "y")
        check(lib().moe_fc2_combine(self._h, ptr(y), stream_ptr(stream)))
        return y

    def backward(self, dy: torch.Tensor, dx=None, dw1=None, dw2=None, dwr=None, want_weight_grads=True,
                 dx_event: "torch.cuda.Event | None" = None, stream=None):
        """dx first (fc2 dgrad + SwiGLU bwd, fc1 dgrad + gather, combine), then
        the weight gradients; `dx_event` is recorded as soon as dx is final."""
        require_cuda(dy)
        dy = _check(dy.contiguous(), (self.Tr, self.h), torch.bfloat16, "dy")
        if dx is None:
            dx = torch.empty(self.Tr, self.h, dtype=torch.bfloat16, device="cuda")
        if want_weight_grads:
            if dw1 is None:
                dw1 = torch.empty(self.el, 2 * self.f, self.h, dtype=torch.bfloat16, device="cuda")
            if dw2 is None:
                dw2 = torch.empty(self.el, self.h, self.f, dtype=torch.bfloat16, device="cuda")
            if dwr is None:
                dwr = torch.empty(self.E, self.h, dtype=torch.float32, device="cuda")
        _check(dx, (self.Tr, self.h), torch.bfloat16, "dx")
        _check(dw1, (self.el, 2 * self.f, self.h), torch.bfloat16, "dw1")
        _check(dw2, (self.el, self.h, self.f), torch.bfloat16, "dw2")
        _check(dwr, (self.E, self.h), torch.float32, "dwr")
        ev = C.c_void_p(dx_event.cuda_event) if dx_event is not None else C.c_void_p(None)
        check(lib().moe_layer_backward_ex(self._h, ptr(dy), ptr(dx), ptr(dw1), ptr(dw2), ptr(dwr), ev,
                                          stream_ptr(stream)))
        return dx, dw1, dw2, dwr

    def routing(self):
        """Routing results of the last forward (device tensors)."""
        v = _RoutingView()
        check(lib().moe_layer_routing(self._h, C.byref(v)))
        T = self.Tr * self.n
        torch.cuda.synchronize()
        rows = int(_view(v.rows, (1,), torch.int32).item())
        return dict(
            experts=_view(v.experts, (T, self.k), torch.int32),
            gates=_view(v.gates, (T, self.k), torch.float32),
            dropped=_view(v.dropped, (T,), torch.uint8),
            row_map_in=_view(v.row_map_in, (max(rows, 1),), torch.int32)[:rows],
            per_expert_counts=_view(v.per_expert_counts, (self.E,), torch.int32),
            out_expert=_view(v.out_expert, (max(rows, 1),), torch.int32)[:rows],
            out_source_rank=_view(v.out_source_rank, (max(rows, 1),), torch.int32)[:rows],
            dgates=_view(v.dgates, (self.Tr, self.k), torch.float32),
            logits=_view(v.logits, (self.Tr, self.E), torch.float32),
        )

    def enable_timing(self, on=True):
        check(lib().moe_layer_enable_timing(self._h, int(on)))

    def phase_times(self):
        ms = (C.c_float * 32)()
        names = (C.c_char_p * 32)()
        cnt = C.c_int()
        check(lib().moe_layer_phase_times(self._h, ms, 32, C.byref(cnt), names))
        return {names[i].decode(): ms[i] for i in range(cnt.value)}

    def enable_stamps(self, on=True):
        """%globaltimer stamps at phase boundaries and barrier entry/release
        (captured into CUDA graphs; see moe_layer_enable_stamps)."""
        check(lib().moe_layer_enable_stamps(self._h, int(bool(on))))

    def read_stamps(self):
        """(phase -> ns, barrier slot -> (entry ns, release ns)) of the last step."""
        buf = (C.c_uint64 * 64)()
        names = (C.c_char_p * 64)()
        cnt = C.c_int()
        check(lib().moe_layer_read_stamps(self._h, buf, 64, C.byref(cnt), names))
        n = cnt.value
        phases = {names[i].decode(): int(buf[i]) for i in range(n) if buf[i]}
        bars = {s: (int(buf[n + 2 * s]), int(buf[n + 2 * s + 1])) for s in range(4) if buf[n + 2 * s]}
        return phases, bars

    def set_fused_dispatch(self, on: bool):
        check(lib().moe_layer_set_fused_dispatch(self._h, int(bool(on))))

    def fused_dispatch(self) -> bool:
        return bool(lib().moe_layer_get_fused_dispatch(self._h))

    def set_compute_only(self, on: bool):
        """Exposed-comm measurement mode (see moe_layer_set_comm_mode)."""
        check(lib().moe_layer_set_comm_mode(self._h, int(bool(on))))

    def error_flag(self) -> int:
        return int(lib().moe_layer_error_flag(self._h))

    def status(self, stream=None) -> None:
        """Synchronise and raise MoETimeout if a cross-GPU wait gave up."""
        check(lib().moe_layer_status(self._h, stream_ptr(stream)))

    def clear_error(self) -> None:
        check(lib().moe_layer_clear_error(self._h))

    # ------------------------------------------------------------------
    def connect(self, group=None):
        """Exchange IPC handles with every rank (collective over torch.distributed)."""
        from .dist import exchange_blobs
        sz = int(lib().moe_layer_ipc_handle_size())
        blob = (C.c_uint8 * sz)()
        check(lib().moe_layer_ipc_export(self._h, blob))
        joined = exchange_blobs(bytes(blob), self.n, group)
        buf = (C.c_uint8 * len(joined)).from_buffer_copy(joined)
        check(lib().moe_layer_ipc_import(self._h, buf))
