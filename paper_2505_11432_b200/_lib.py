"""ctypes binding of libmoe_b200.so (the C ABI in include/moe_b200.h).

The product path has no fallback: if the CUDA library is missing or cannot
be loaded, every operator raises. Torch is used only for device memory and
streams (tensors are passed as raw pointers).
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmoe_b200.so")

MOE_OK, MOE_ERR_INTERNAL, MOE_ERR_INVALID, MOE_ERR_CUDA, MOE_ERR_TIMEOUT, MOE_ERR_UNSUPPORTED = range(6)


class MoEError(RuntimeError):
    """Non-domain failure (reference: std::exception -> exit 1)."""


class DomainError(ValueError):
    """Invalid argument (reference: std::domain_error -> exit 2)."""


class MoETimeout(MoEError):
    pass


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise MoEError(f"{LIB_PATH} not built: run `make` (or __graft_entry__.build()); "
                           "there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        L.moe_last_error.restype = C.c_char_p
        L.moe_launch_count.restype = C.c_uint64
        L.moe_permute_workspace_size.restype = C.c_size_t
        L.moe_permute_workspace_size.argtypes = [C.c_int64] * 4
        for name, res, args in (("moe_layer_input_buffer", C.c_void_p, [C.c_void_p]),
                                ("moe_layer_dy_buffer", C.c_void_p, [C.c_void_p]),
                                ("moe_layer_ipc_handle_size", C.c_size_t, []),
                                ("moe_layer_destroy", None, [C.c_void_p])):
            if hasattr(L, name):
                getattr(L, name).restype = res
                getattr(L, name).argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == MOE_OK:
        return
    msg = lib().moe_last_error().decode(errors="replace")
    if status == MOE_ERR_INVALID:
        raise DomainError(msg)
    if status == MOE_ERR_TIMEOUT:
        raise MoETimeout(msg)
    raise MoEError(f"status {status}: {msg}")


def ptr(t) -> C.c_void_p:
    if t is None:
        return C.c_void_p(None)
    if isinstance(t, int):
        return C.c_void_p(t)
    return C.c_void_p(t.data_ptr())


def stream_ptr(stream=None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def i64(v) -> C.c_int64:
    return C.c_int64(int(v))


def launch_count() -> int:
    return int(lib().moe_launch_count())


def launch_count_reset() -> None:
    lib().moe_launch_count_reset()


def require_cuda(*tensors) -> None:
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise DomainError("tensor must live on a CUDA device (no CPU fallback)")
