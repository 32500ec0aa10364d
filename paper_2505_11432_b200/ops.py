"""Thin operator wrappers over the C ABI for the dense pieces of the hot
path: the tcgen05 grouped GEMM (reference OpKind::grouped_gemm,
simsched.hpp:32-44) and the FP8 per-token quantiser (numerics.hpp:61-62)."""
from __future__ import annotations

import torch

from ._lib import DomainError, check, i64, lib, ptr, require_cuda, stream_ptr


def grouped_gemm(a: torch.Tensor, b: torch.Tensor, group_rows: torch.Tensor, *, N: int, K: int,
                 M: int = 0, a_mn_major=False, b_mn_major=False, k_grouped=False,
                 out_dtype=torch.bfloat16, bn=256, cta_pair=False, out=None, stream=None) -> torch.Tensor:
    """M-grouped: a [rows, K] (K-major), b [G*N, K] (K-major) or [G*K, N]
    (MN-major) -> out [rows, N]; group g owns group_rows[g] rows (multiple
    of 128; with cta_pair a trailing 128-row block runs as an M=128 pair tile). K-grouped: a [rows, M], b [rows, N] (both MN-major) ->
    out [G*M, N], out_g = a_g^T b_g."""
    require_cuda(a, b, group_rows)
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise DomainError("grouped_gemm takes bf16 operands")
    G = int(group_rows.shape[0])
    rows = int(a.shape[0])
    if out is None:
        shape = (G * M, N) if k_grouped else (rows, N)
        out = torch.empty(shape, dtype=out_dtype, device=a.device)
    check(lib().moe_grouped_gemm(ptr(a), ptr(b), ptr(out), G, ptr(group_rows), i64(rows), i64(M),
                                 i64(N), i64(K), int(a_mn_major), int(b_mn_major), int(k_grouped),
                                 int(out.dtype == torch.float32), int(bn), int(bool(cta_pair)),
                                 stream_ptr(stream)))
    return out


def quantize_e4m3_rows(x: torch.Tensor, stream=None):
    """Per-token E4M3: codes (uint8 bits) [rows, cols], fp32 scales [rows]."""
    require_cuda(x)
    rows, cols = x.shape
    codes = torch.empty(rows, cols, dtype=torch.uint8, device=x.device)
    scales = torch.empty(rows, dtype=torch.float32, device=x.device)
    x = x.contiguous()
    if x.dtype == torch.float32:
        check(lib().moe_quantize_e4m3_rows_f32(ptr(x), i64(rows), i64(cols), ptr(codes), ptr(scales), stream_ptr(stream)))
    elif x.dtype == torch.bfloat16:
        check(lib().moe_quantize_e4m3_rows(ptr(x), i64(rows), i64(cols), ptr(codes), ptr(scales), stream_ptr(stream)))
    else:
        raise DomainError("quantize takes fp32 or bf16")
    return codes, scales


def ffn_forward_f32(x: torch.Tensor, w1: torch.Tensor, w2: torch.Tensor, wr: torch.Tensor | None, k: int,
                    capacity_factor: float = 0.0, gate_order: str = "before_fc2_in", experts=None, gates=None,
                    stream=None):
    """fp32 MoE layer forward (configs[0]); returns y, experts, gates, logits, dropped."""
    import ctypes as C
    require_cuda(x, w1, w2)
    T, h = x.shape
    E, f2, _ = w1.shape
    dev = x.device
    y = torch.empty(T, h, dtype=torch.float32, device=dev)
    ex = torch.empty(T, k, dtype=torch.int32, device=dev)
    g = torch.empty(T, k, dtype=torch.float32, device=dev)
    lg = torch.empty(T, E, dtype=torch.float32, device=dev)
    dr = torch.empty(T, dtype=torch.uint8, device=dev)
    check(lib().moe_ffn_forward_f32(ptr(x.contiguous()), ptr(w1.contiguous()), ptr(w2.contiguous()),
                                    ptr(None if wr is None else wr.contiguous()), i64(T), i64(h), i64(f2 // 2),
                                    i64(E), i64(k), C.c_double(capacity_factor),
                                    int(gate_order.startswith("after")), ptr(experts), ptr(gates), ptr(y),
                                    ptr(ex), ptr(g), ptr(lg), ptr(dr), stream_ptr(stream)))
    return y, ex, g, lg, dr


def quantize_e4m3_fast(x: torch.Tensor, group: int = 0, stream=None):
    """The layer's dispatch-payload quantiser: bf16 [rows, cols] -> E4M3 codes
    (uint8 bits) + fp32 scales; group 0 = per-token (scales [rows]), 128 =
    grouped-128 (scales [rows, cols/128])."""
    require_cuda(x)
    if x.dtype != torch.bfloat16 or x.dim() != 2:
        raise DomainError("quantize_e4m3_fast takes a bf16 [rows, cols] tensor")
    rows, cols = x.shape
    codes = torch.empty(rows, cols, dtype=torch.uint8, device=x.device)
    scales = torch.empty((rows,) if group == 0 else (rows, cols // 128), dtype=torch.float32, device=x.device)
    check(lib().moe_quantize_e4m3_fast(ptr(x.contiguous()), i64(rows), i64(cols), int(group), ptr(codes),
                                       ptr(scales), stream_ptr(stream)))
    return codes, scales


def grouped_gemm_e4m3(a: torch.Tensor, b: torch.Tensor, group_rows: torch.Tensor, *, N: int, K: int,
                      b_mn_major=False, cta_pair=False, stream=None):
    """M-grouped GEMM whose epilogue quantises the fp32 accumulators
    grouped-128 to E4M3 (the fc2 / fc1-dgrad FP8 combine payload):
    codes [rows, N] uint8 + scales [rows, N/128] fp32."""
    require_cuda(a, b, group_rows)
    rows = int(a.shape[0])
    codes = torch.empty(rows, N, dtype=torch.uint8, device=a.device)
    scales = torch.empty(rows, N // 128, dtype=torch.float32, device=a.device)
    check(lib().moe_grouped_gemm_e4m3(ptr(a), ptr(b), ptr(codes), ptr(scales), int(group_rows.shape[0]),
                                      ptr(group_rows), i64(rows), i64(N), i64(K), int(bool(b_mn_major)),
                                      int(bool(cta_pair)), stream_ptr(stream)))
    return codes, scales
