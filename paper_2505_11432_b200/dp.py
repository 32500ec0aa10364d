"""Data-parallel gradient synchronisation with BF16 communication compression
(reference cost model commcost.cpp:182-201 `dp_sync_time`
with compressed = true, memory model memmodel.cpp:112-114): an in-place
bf16 all-to-all reduce-scatter with binary64/fp32 local reduction, and a
bf16 all-gather (C ABI moe_dp_*)."""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import DomainError, check, i64, lib, ptr, require_cuda, stream_ptr
from .layer import _view


class DpGradSync:
    def __init__(self, count: int, dp_size: int = 1, rank: int = 0):
        L = lib()
        for name in ("moe_dp_grad_buffer", "moe_dp_shard"):
            getattr(L, name).restype = C.c_void_p
            getattr(L, name).argtypes = [C.c_void_p]
        L.moe_dp_destroy.argtypes = [C.c_void_p]
        L.moe_dp_destroy.restype = None
        L.moe_dp_ipc_handle_size.restype = C.c_size_t
        self.count, self.n, self.rank = count, dp_size, rank
        self.shard_size = count // dp_size
        h_ = C.c_void_p()
        check(L.moe_dp_create(i64(count), i64(dp_size), i64(rank), C.byref(h_)))
        self._h = h_
        self.grad = _view(L.moe_dp_grad_buffer(h_), (count,), torch.float32)
        self.shard = _view(L.moe_dp_shard(h_), (self.shard_size,), torch.float32)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().moe_dp_destroy(h)
            self._h = None

    def connect(self, group=None):
        from .dist import exchange_blobs
        sz = int(lib().moe_dp_ipc_handle_size())
        blob = (C.c_uint8 * sz)()
        check(lib().moe_dp_ipc_export(self._h, blob))
        joined = exchange_blobs(bytes(blob), self.n, group)
        check(lib().moe_dp_ipc_import(self._h, (C.c_uint8 * len(joined)).from_buffer_copy(joined)))

    def reduce_scatter(self, stream=None) -> torch.Tensor:
        """Consumes `self.grad`; returns this rank's reduced fp32 shard (a view
        into the same buffer)."""
        check(lib().moe_dp_reduce_scatter(self._h, stream_ptr(stream)))
        return self.shard

    def all_gather_bf16(self, shard: torch.Tensor, out=None, stream=None) -> torch.Tensor:
        require_cuda(shard)
        if shard.dtype != torch.float32 or shard.numel() != self.shard_size:
            raise DomainError("shard must be fp32 [count / dp_size]")
        if out is None:
            out = torch.empty(self.count, dtype=torch.bfloat16, device="cuda")
        check(lib().moe_dp_all_gather_bf16(self._h, ptr(shard.contiguous()), ptr(out), stream_ptr(stream)))
        return out

    def error_flag(self) -> int:
        return int(lib().moe_dp_error_flag(self._h))

    def status(self, stream=None) -> None:
        """Synchronise and raise MoETimeout if a cross-GPU wait gave up."""
        check(lib().moe_dp_status(self._h, stream_ptr(stream)))
