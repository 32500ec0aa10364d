"""Ulysses sequence-parallel attention projections (PAPER.md:150-160,
294-302; reference AttnStrategy::sp nodes qkv_proj -> a2a_qkv and
a2a_attn_out -> out_proj, graph.cpp:189-201): fused GEMM+A2A and A2A+GEMM
over NVLink (C ABI moe_ulysses_*)."""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import DomainError, check, i64, lib, ptr, require_cuda, stream_ptr
from .layer import _view


class UlyssesProjections:
    def __init__(self, seq: int, hidden: int, qkv_cols: int, sp_size: int = 1, rank: int = 0):
        L = lib()
        for name in ("moe_ulysses_qkv_buffer", "moe_ulysses_attn_out_buffer"):
            getattr(L, name).restype = C.c_void_p
            getattr(L, name).argtypes = [C.c_void_p]
        L.moe_ulysses_destroy.argtypes = [C.c_void_p]
        L.moe_ulysses_destroy.restype = None
        L.moe_ulysses_ipc_handle_size.restype = C.c_size_t
        self.s, self.h, self.nqkv, self.n, self.rank = seq, hidden, qkv_cols, sp_size, rank
        self.sr, self.cpo, self.dh = seq // sp_size, qkv_cols // sp_size, hidden // sp_size
        h_ = C.c_void_p()
        check(L.moe_ulysses_create(i64(seq), i64(hidden), i64(qkv_cols), i64(sp_size), i64(rank), C.byref(h_)))
        self._h = h_
        self.qkv_heads = _view(L.moe_ulysses_qkv_buffer(h_), (seq, self.cpo), torch.bfloat16)
        self.attn_out = _view(L.moe_ulysses_attn_out_buffer(h_), (seq, self.dh), torch.bfloat16)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().moe_ulysses_destroy(h)
            self._h = None

    def set_weights(self, wqkv: torch.Tensor, wout: torch.Tensor, stream=None):
        """wqkv [qkv_cols, h] (rows ordered by owning rank), wout [h, h], bf16."""
        require_cuda(wqkv, wout)
        if wqkv.shape != (self.nqkv, self.h) or wout.shape != (self.h, self.h):
            raise DomainError("weights must be wqkv [qkv_cols, h] and wout [h, h]")
        self._keep = (wqkv.contiguous(), wout.contiguous())
        check(lib().moe_ulysses_set_weights(self._h, ptr(self._keep[0]), ptr(self._keep[1]), stream_ptr(stream)))

    def connect(self, group=None):
        from .dist import exchange_blobs
        sz = int(lib().moe_ulysses_ipc_handle_size())
        blob = (C.c_uint8 * sz)()
        check(lib().moe_ulysses_ipc_export(self._h, blob))
        joined = exchange_blobs(bytes(blob), self.n, group)
        check(lib().moe_ulysses_ipc_import(self._h, (C.c_uint8 * len(joined)).from_buffer_copy(joined)))

    def qkv_a2a(self, x_shard: torch.Tensor, stream=None) -> torch.Tensor:
        """GEMM + A2A; returns the [s, qkv_cols/sp] head-group buffer (valid
        until the next call)."""
        require_cuda(x_shard)
        if x_shard.shape != (self.sr, self.h):
            raise DomainError("x_shard must be [s/sp, h]")
        self._x = x_shard.contiguous()
        check(lib().moe_ulysses_qkv_a2a(self._h, ptr(self._x), stream_ptr(stream)))
        return self.qkv_heads

    def a2a_out_proj(self, o_heads=None, out=None, stream=None) -> torch.Tensor:
        if o_heads is not None:
            require_cuda(o_heads)
        if out is None:
            out = torch.empty(self.sr, self.h, dtype=torch.bfloat16, device="cuda")
        check(lib().moe_ulysses_a2a_out_proj(self._h, ptr(None if o_heads is None else o_heads.contiguous()),
                                             ptr(out), stream_ptr(stream)))
        return out

    def error_flag(self) -> int:
        return int(lib().moe_ulysses_error_flag(self._h))

    def status(self, stream=None) -> None:
        """Synchronise and raise MoETimeout if a cross-GPU wait gave up."""
        check(lib().moe_ulysses_status(self._h, stream_ptr(stream)))
