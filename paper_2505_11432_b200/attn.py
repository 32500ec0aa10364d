"""Sequence-parallel attention projections with tensor-parallel weights
(reference nodes ag_attn_in -> qkv_proj and out_proj -> rs_attn_out,
graph.cpp:202-214): fused AG-GEMM and GEMM-RS over NVLink (C ABI
moe_attn_*)."""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import DomainError, check, i64, lib, ptr, require_cuda, stream_ptr
from .layer import _view


class AttnProjections:
    def __init__(self, seq: int, hidden: int, qkv_cols_per_rank: int, tp_size: int = 1, rank: int = 0):
        L = lib()
        L.moe_attn_input_buffer.restype = C.c_void_p
        L.moe_attn_input_buffer.argtypes = [C.c_void_p]
        L.moe_attn_destroy.argtypes = [C.c_void_p]
        L.moe_attn_destroy.restype = None
        L.moe_attn_ipc_handle_size.restype = C.c_size_t
        self.s, self.h, self.nq, self.n, self.rank = seq, hidden, qkv_cols_per_rank, tp_size, rank
        self.sr, self.dh = seq // tp_size, hidden // tp_size
        h_ = C.c_void_p()
        check(L.moe_attn_create(i64(seq), i64(hidden), i64(qkv_cols_per_rank), i64(tp_size), i64(rank),
                                C.byref(h_)))
        self._h = h_
        self.input_buffer = _view(L.moe_attn_input_buffer(h_), (self.sr, hidden), torch.bfloat16)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().moe_attn_destroy(h)
            self._h = None

    def set_weights(self, wqkv: torch.Tensor, wout: torch.Tensor, stream=None):
        """wqkv [qkv_cols_per_rank, h], wout [h, h/tp] (nn.Linear layout), bf16."""
        require_cuda(wqkv, wout)
        if wqkv.shape != (self.nq, self.h) or wout.shape != (self.h, self.dh):
            raise DomainError("weights must be wqkv [qkv_cols, h] and wout [h, h/tp]")
        self._keep = (wqkv.contiguous(), wout.contiguous())
        check(lib().moe_attn_set_weights(self._h, ptr(self._keep[0]), ptr(self._keep[1]), stream_ptr(stream)))

    def connect(self, group=None):
        from .dist import exchange_blobs
        sz = int(lib().moe_attn_ipc_handle_size())
        blob = (C.c_uint8 * sz)()
        check(lib().moe_attn_ipc_export(self._h, blob))
        joined = exchange_blobs(bytes(blob), self.n, group)
        check(lib().moe_attn_ipc_import(self._h, (C.c_uint8 * len(joined)).from_buffer_copy(joined)))

    def ag_gemm(self, x_shard=None, out=None, stream=None):
        if out is None:
            out = torch.empty(self.s, self.nq, dtype=torch.bfloat16, device="cuda")
        check(lib().moe_attn_ag_gemm(self._h, ptr(x_shard), ptr(out), stream_ptr(stream)))
        return out

    def gemm_rs(self, o: torch.Tensor, out=None, stream=None):
        require_cuda(o)
        if out is None:
            out = torch.empty(self.sr, self.h, dtype=torch.bfloat16, device="cuda")
        check(lib().moe_attn_gemm_rs(self._h, ptr(o.contiguous()), ptr(out), stream_ptr(stream)))
        return out

    def error_flag(self) -> int:
        return int(lib().moe_attn_error_flag(self._h))

    def status(self, stream=None) -> None:
        """Synchronise and raise MoETimeout if a cross-GPU wait gave up."""
        check(lib().moe_attn_status(self._h, stream_ptr(stream)))
