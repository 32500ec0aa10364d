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
    of 128, or of 256 with cta_pair). K-grouped: a [rows, M], b [rows, N] (both MN-major) ->
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
