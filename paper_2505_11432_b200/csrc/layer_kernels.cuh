// layer_kernels.cuh — the memory-bound operators of the MoE layer around
// the grouped GEMMs: permuted-row metadata, dispatch (AG + local scatter),
// combine (gather + reduce), SwiGLU/gate backward reductions, router
// backward, weight packing and the cross-GPU flag barrier.
//
// Reference operator nodes (graph.cpp): scatter :276-286, gather :302-306,
// weighted_sum :292-295, router :268-271, collectives ag_ffn_in/rs_ffn_out
// :276-310. All of these are HBM- or NVLink-bound; kernels use 16-byte
// vector accesses, one warp per row, grids sized to the SM count.
#pragma once

#include "common.cuh"
#include "topk.cuh"

namespace moe {

// Per padded permuted row: source token-slot, gate, combine destination.
// Grid: one block per local expert.
static __global__ void row_info_kernel(const int32_t* __restrict__ group_pad_off,
                                const int32_t* __restrict__ group_pad_rows,
                                const int32_t* __restrict__ expert_offsets,
                                int32_t* __restrict__ pad_row_tok,  // in: real rows; out: -1 pads
                                const float* __restrict__ gates_all, int k, int tokens_per_rank,
                                float* __restrict__ row_gate, int32_t* __restrict__ row_dst) {
    const int g = blockIdx.x;
    const int poff = group_pad_off[g], pr = group_pad_rows[g];
    const int cnt = expert_offsets[g + 1] - expert_offsets[g];
    for (int r = threadIdx.x; r < pr; r += blockDim.x) {
        const int pp = poff + r;
        if (r < cnt) {
            const int i = pad_row_tok[pp];  // t*k + slot (global token id)
            const int t = i / k, slot = i - t * k;
            const int src = t / tokens_per_rank;
            row_gate[pp] = gates_all[i];
            row_dst[pp] = (src << 27) | ((t - src * tokens_per_rank) * k + slot);
        } else {
            pad_row_tok[pp] = -1;
            row_gate[pp] = 0.0f;
            row_dst[pp] = -1;
        }
    }
}

// Dispatch dedup: the first padded row of every token on this rank
// (first_row pre-filled with 0x7f7f7f7f), then every later row of the same
// token points at it (its k experts on one rank need the token row once).
static __global__ void first_row_kernel(const int32_t* __restrict__ pad_row_tok, const int32_t* nrows_pad, int k,
                                        int32_t* __restrict__ first_row) {
    const int total = *nrows_pad;
    for (int pp = blockIdx.x * blockDim.x + threadIdx.x; pp < total; pp += gridDim.x * blockDim.x) {
        const int i = pad_row_tok[pp];
        if (i >= 0) atomicMin(&first_row[i / k], pp);
    }
}
static __global__ void dup_src_kernel(const int32_t* __restrict__ pad_row_tok, const int32_t* nrows_pad, int k,
                                      const int32_t* __restrict__ first_row, int32_t* __restrict__ dup_src) {
    const int total = *nrows_pad;
    for (int pp = blockIdx.x * blockDim.x + threadIdx.x; pp < total; pp += gridDim.x * blockDim.x) {
        const int i = pad_row_tok[pp];
        const int f = i >= 0 ? first_row[i / k] : pp;
        dup_src[pp] = f != pp ? f : -1;
    }
}

// Dispatch: dst[pp, :] = src_rank_buffer[t_local, :] for real rows, 0 for
// pads (AG + local scatter fused: rows are pulled straight from the owning
// rank's buffer over NVLink into permuted order).
// One warp per row, 16-byte vectors, 16 in flight per lane.
static __global__ void dispatch_rows_kernel(const int32_t* __restrict__ pad_row_tok, const int32_t* nrows_pad,
                                     int k, int tokens_per_rank, int h,
                                     const uint16_t* const* __restrict__ src_bufs,
                                     uint16_t* __restrict__ dst) {
    // (unfused reference path: bf16 only, no row scaling)
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int total = *nrows_pad;
    const int nvec = h / 8;
    for (int pp = warp; pp < total; pp += nwarps) {
        const int i = pad_row_tok[pp];
        uint4* d = reinterpret_cast<uint4*>(dst + (int64_t)pp * h);
        if (i < 0) {
            for (int v = lane; v < nvec; v += 32) d[v] = make_uint4(0, 0, 0, 0);
            continue;
        }
        const int t = i / k;
        const int src = t / tokens_per_rank;
        const uint4* s = reinterpret_cast<const uint4*>(src_bufs[src] + (int64_t)(t - src * tokens_per_rank) * h);
        // 16 x 16 B loads in flight per lane (a whole 4096-wide row), predicated tail
        constexpr int U = 16;
        for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
            uint4 r[U];
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (v0 + 32 * q < nvec) r[q] = s[v0 + 32 * q];
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (v0 + 32 * q < nvec) d[v0 + 32 * q] = r[q];
        }
    }
}

// Router backward helper: given gates g (softmax over the k selected logits)
// and dgates, dlogit_j = g_j (dg_j - sum_i g_i dg_i).
__device__ __forceinline__ void softmax_topk_bwd(const float* g, const float* dg, int k, float* dl) {
    float s = 0.0f;
    for (int j = 0; j < k; ++j) s += g[j] * dg[j];
    for (int j = 0; j < k; ++j) dl[j] = g[j] * (dg[j] - s);
}

// Combine: y[t, :] = sum over slots (fixed slot order, fp32) of the staged
// expert outputs (a2a_fp32 semantics, numerics.cpp:172-192); dropped tokens
// produce 0. FP8 = staged rows are grouped-128 E4M3 codes + fp32 scales
// (dequantised on arrival). slot_gate (gate after fc2, numerics.hpp:84-86)
// multiplies each slot. Optional router term for dx:
// += sum_j dlogit_j * wr[e_j, :]. One warp per token; lanes own 16 columns.
template <bool FP8, int KT = 0>   // KT: compile-time slot count (0 = runtime k)
static __global__ void combine_reduce_kernel(const void* __restrict__ stage_v, const float* __restrict__ stage_scale,
                                      const uint8_t* __restrict__ dropped, int T, int k, int h,
                                      uint16_t* __restrict__ out, const float* __restrict__ slot_gate,
                                      const int32_t* __restrict__ experts, const float* __restrict__ gates,
                                      const float* __restrict__ dgates, const uint16_t* __restrict__ wr,
                                      float* __restrict__ dlogits, int E) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int nv16 = h / 16;
    const int kk = KT > 0 ? KT : k;
    for (int t = warp; t < T; t += nwarps) {
        uint4* o = reinterpret_cast<uint4*>(out + (int64_t)t * h);
        if (dropped && dropped[t]) {
            for (int v = lane; v < h / 8; v += 32) o[v] = make_uint4(0, 0, 0, 0);
            if (dlogits) for (int e = lane; e < E; e += 32) dlogits[(int64_t)t * E + e] = 0.0f;
            continue;
        }
        float dl[8];
        int ex[8];
        float sg[8];
        const bool router = wr != nullptr;
#pragma unroll
        for (int j = 0; j < kk; ++j) sg[j] = slot_gate ? slot_gate[(int64_t)t * kk + j] : 1.0f;
        if (router) {
            float g[8], dg[8];
#pragma unroll
            for (int j = 0; j < kk; ++j) {
                g[j] = gates[(int64_t)t * kk + j];
                dg[j] = dgates[(int64_t)t * kk + j];
                ex[j] = experts[(int64_t)t * kk + j];
            }
            softmax_topk_bwd(g, dg, kk, dl);
            if (dlogits) {
                for (int e = lane; e < E; e += 32) {
                    float v = 0.0f;
#pragma unroll
                    for (int j = 0; j < kk; ++j) v = (ex[j] == e) ? dl[j] : v;
                    dlogits[(int64_t)t * E + e] = v;
                }
            }
        }
#pragma unroll 2
        for (int v = lane; v < nv16; v += 32) {
            float acc[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] = 0.0f;
#pragma unroll
            for (int j = 0; j < kk; ++j) {
                const int64_t row = (int64_t)t * kk + j;
                if (FP8) {
                    const uint4 c = reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(stage_v) + row * h)[v];
                    const float f = stage_scale[row * (h / 128) + (v * 16) / 128] * sg[j];
                    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float2 lo = e4m3x2_to_f32x2((uint16_t)(w[q] & 0xffff));
                        const float2 hi = e4m3x2_to_f32x2((uint16_t)(w[q] >> 16));
                        acc[4 * q] += lo.x * f; acc[4 * q + 1] += lo.y * f;
                        acc[4 * q + 2] += hi.x * f; acc[4 * q + 3] += hi.y * f;
                    }
                } else {
                    const uint4* sp = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(stage_v) + row * h);
                    const uint4 s0 = sp[2 * v], s1 = sp[2 * v + 1];
                    const uint32_t w[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float2 p = unpack_bf16x2(w[q]);
                        acc[2 * q] += p.x * sg[j];
                        acc[2 * q + 1] += p.y * sg[j];
                    }
                }
            }
            if (router) {
#pragma unroll
                for (int j = 0; j < kk; ++j) {
                    const uint4* wp = reinterpret_cast<const uint4*>(wr + (int64_t)ex[j] * h);
                    const uint4 w0 = wp[2 * v], w1 = wp[2 * v + 1];
                    const uint32_t w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float2 p = unpack_bf16x2(w[q]);
                        acc[2 * q] += dl[j] * p.x;
                        acc[2 * q + 1] += dl[j] * p.y;
                    }
                }
            }
            o[2 * v] = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                                  pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
            o[2 * v + 1] = make_uint4(pack_bf16x2(acc[8], acc[9]), pack_bf16x2(acc[10], acc[11]),
                                      pack_bf16x2(acc[12], acc[13]), pack_bf16x2(acc[14], acc[15]));
        }
    }
}

// Host launcher: compile-time slot count for k <= 4 (all loads of a column
// block unrolled: Mixtral combine_dx 23 -> 18.5 us), runtime k otherwise.
template <bool FP8>
static void launch_combine(cudaStream_t st, const void* stage_v, const float* stage_scale, const uint8_t* dropped,
                           int T, int k, int h, uint16_t* out, const float* slot_gate, const int32_t* experts,
                           const float* gates, const float* dgates, const uint16_t* wr, float* dlogits, int E) {
    const dim3 grid(kNumSMs * 4), block(256);
#define MOE_COMBINE(KT) \
    combine_reduce_kernel<FP8, KT><<<grid, block, 0, st>>>(stage_v, stage_scale, dropped, T, k, h, out, slot_gate, \
                                                           experts, gates, dgates, wr, dlogits, E)
    switch (k) {
        case 1: MOE_COMBINE(1); break;
        case 2: MOE_COMBINE(2); break;
        case 4: MOE_COMBINE(4); break;
        default: MOE_COMBINE(0); break;   // k = 8 unrolled measured slower (116 regs)
    }
#undef MOE_COMBINE
}

// Gate-after-fc2 backward on the source rank (numerics.hpp:84-86):
// dgate[t, j] = <dy[t, :], fc2_out[t, j, :]> with fc2_out the pre-gate expert
// output still held in this rank's combine staging from the forward pass.
template <bool FP8>
static __global__ void dgate_after_kernel(const uint16_t* __restrict__ dy, const void* __restrict__ stage_v,
                                   const float* __restrict__ stage_scale, const uint8_t* __restrict__ dropped,
                                   int T, int k, int h, float* __restrict__ dgate) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int t = warp; t < T; t += nwarps) {
        const bool drop = dropped && dropped[t];
        for (int j = 0; j < k; ++j) {
            const int64_t row = (int64_t)t * k + j;
            float acc = 0.0f;
            if (!drop) {
                for (int v = lane; v < h / 16; v += 32) {
                    const uint4* dp = reinterpret_cast<const uint4*>(dy + (int64_t)t * h);
                    const uint4 d0 = dp[2 * v], d1 = dp[2 * v + 1];
                    const uint32_t dw[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
                    float sv[16];
                    if (FP8) {
                        const uint4 c = reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(stage_v) + row * h)[v];
                        const float f = stage_scale[row * (h / 128) + (v * 16) / 128];
                        const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float2 lo = e4m3x2_to_f32x2((uint16_t)(w[q] & 0xffff));
                            const float2 hi = e4m3x2_to_f32x2((uint16_t)(w[q] >> 16));
                            sv[4 * q] = lo.x * f; sv[4 * q + 1] = lo.y * f;
                            sv[4 * q + 2] = hi.x * f; sv[4 * q + 3] = hi.y * f;
                        }
                    } else {
                        const uint4* sp = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(stage_v) + row * h);
                        const uint4 s0 = sp[2 * v], s1 = sp[2 * v + 1];
                        const uint32_t w[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float2 p = unpack_bf16x2(w[q]);
                            sv[2 * q] = p.x;
                            sv[2 * q + 1] = p.y;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float2 d = unpack_bf16x2(dw[q]);
                        acc += d.x * sv[2 * q] + d.y * sv[2 * q + 1];
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            }
            if (lane == 0) dgate[row] = drop ? 0.0f : acc;
        }
    }
}

// Source-side E4M3 quantisation of this rank's rows before they are pulled
// over NVLink (FP8 communication): GROUP = 0 -> one scale
// per row (per_token, forward), else one per GROUP columns (grouped-128,
// backward). Codes bit-identical to the reference quantize (binary64
// x / scale, numerics.cpp:149-156) through e4m3_block / e4m3x2_code
// (common.cuh): fp32 fast path, binary64 division near rounding midpoints.
template <int GROUP>
static __global__ void quantize_fast_kernel(const uint16_t* __restrict__ x, int rows, int cols,
                                     uint8_t* __restrict__ codes, float* __restrict__ scales) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int r = warp; r < rows; r += nwarps) {
        const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)r * cols);
        if (GROUP == 0) {
            float m = 0.0f;
            for (int v = lane; v < cols / 8; v += 32) {
                const uint4 a = xr[v];
                const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 p = unpack_bf16x2(w[q]);
                    m = fmaxf(m, fmaxf(fabsf(p.x), fabsf(p.y)));
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
            const E4m3Block blk = e4m3_block(m);
            if (lane == 0) scales[r] = (float)blk.scale;
            for (int v = lane; v < cols / 8; v += 32) {
                const uint4 a = xr[v];
                const uint32_t w[4] = {a.x, a.y, a.z, a.w};
                uint32_t pk[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const float2 p0 = unpack_bf16x2(w[2 * q]), p1 = unpack_bf16x2(w[2 * q + 1]);
                    pk[q] = (uint32_t)e4m3x2_code(p0.x, p0.y, blk) |
                            ((uint32_t)e4m3x2_code(p1.x, p1.y, blk) << 16);
                }
                *reinterpret_cast<uint2*>(codes + (int64_t)r * cols + v * 8) = make_uint2(pk[0], pk[1]);
            }
        } else {
            // GROUP/8 lanes per group; lanes exchange within their group
            constexpr int LPG = GROUP / 8;
            for (int v0 = 0; v0 < cols / 8; v0 += 32) {
                const int v = v0 + lane;
                uint4 a = make_uint4(0, 0, 0, 0);
                if (v < cols / 8) a = xr[v];
                const uint32_t w[4] = {a.x, a.y, a.z, a.w};
                float m = 0.0f;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 p = unpack_bf16x2(w[q]);
                    m = fmaxf(m, fmaxf(fabsf(p.x), fabsf(p.y)));
                }
#pragma unroll
                for (int off = LPG / 2; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
                const E4m3Block blk = e4m3_block(m);
                if (v < cols / 8) {
                    if ((lane % LPG) == 0) scales[(int64_t)r * (cols / GROUP) + (v * 8) / GROUP] = (float)blk.scale;
                    uint32_t pk[2];
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const float2 p0 = unpack_bf16x2(w[2 * q]), p1 = unpack_bf16x2(w[2 * q + 1]);
                        pk[q] = (uint32_t)e4m3x2_code(p0.x, p0.y, blk) |
                                ((uint32_t)e4m3x2_code(p1.x, p1.y, blk) << 16);
                    }
                    *reinterpret_cast<uint2*>(codes + (int64_t)r * cols + v * 8) = make_uint2(pk[0], pk[1]);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// ep_pattern = ag_rs (commcost.hpp:81): "gather" then "rs_ffn_out"
// (graph.cpp:302-309). The expert GEMM writes its output rows locally; each
// rank then sums, per token, the rows of the slots it served (fixed slot
// order, fp32) and sends ONE partial row per (token, rank) to the owner's
// staging [T_r, n, h]; the owner adds the partials of the ranks that served
// the token in rank order (a2a_fp32 reduction semantics over ranks,
// numerics.cpp:172-192). Only (token, rank) pairs with a served slot move:
// a sparse reduce-scatter, <= min(k, n) rows per token instead of k.
// ---------------------------------------------------------------------------

// inverse of the padded row map: inv[t*k + slot] = padded row (or -1)
static __global__ void inverse_rows_kernel(const int32_t* __restrict__ pad_row_tok, const int32_t* nrows_pad,
                                           int32_t* __restrict__ inv) {
    const int total = *nrows_pad;
    for (int pp = blockIdx.x * blockDim.x + threadIdx.x; pp < total; pp += gridDim.x * blockDim.x) {
        const int i = pad_row_tok[pp];
        if (i >= 0) inv[i] = pp;
    }
}

// one warp per global token: partial = sum of this rank's slot rows -> owner
static __global__ void gather_rs_kernel(const int32_t* __restrict__ experts, const uint8_t* __restrict__ dropped,
                                        const int32_t* __restrict__ inv, int T, int k, int first, int el,
                                        int tokens_per_rank, int n, int self, int h,
                                        const uint16_t* __restrict__ rows, uint16_t* const* __restrict__ dst) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int nv16 = h / 16;
    for (int t = warp; t < T; t += nwarps) {
        if (dropped[t]) continue;
        int rr[8];
        int nr = 0;
        for (int j = 0; j < k; ++j) {
            const int e = experts[(int64_t)t * k + j] - first;
            if (e >= 0 && e < el) rr[nr++] = inv[(int64_t)t * k + j];
        }
        if (nr == 0) continue;
        const int src = t / tokens_per_rank;
        uint4* o = reinterpret_cast<uint4*>(dst[src] + ((int64_t)(t - src * tokens_per_rank) * n + self) * h);
        for (int v = lane; v < nv16; v += 32) {
            float acc[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] = 0.0f;
            for (int j = 0; j < nr; ++j) {
                const uint4* sp = reinterpret_cast<const uint4*>(rows + (int64_t)rr[j] * h);
                const uint4 s0 = sp[2 * v], s1 = sp[2 * v + 1];
                const uint32_t w[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float2 p = unpack_bf16x2(w[q]);
                    acc[2 * q] += p.x;
                    acc[2 * q + 1] += p.y;
                }
            }
            o[2 * v] = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                                  pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
            o[2 * v + 1] = make_uint4(pack_bf16x2(acc[8], acc[9]), pack_bf16x2(acc[10], acc[11]),
                                      pack_bf16x2(acc[12], acc[13]), pack_bf16x2(acc[14], acc[15]));
        }
    }
}

// owner side: y[t] = sum over the ranks that served t (rank order, fp32) of
// the staged partials; optional router term as in combine_reduce_kernel.
static __global__ void combine_rs_kernel(const uint16_t* __restrict__ stage, const int32_t* __restrict__ experts_loc,
                                         const uint8_t* __restrict__ dropped, int T, int k, int el, int n, int h,
                                         uint16_t* __restrict__ out, const float* __restrict__ gates,
                                         const float* __restrict__ dgates, const uint16_t* __restrict__ wr,
                                         float* __restrict__ dlogits, int E) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int nv16 = h / 16;
    for (int t = warp; t < T; t += nwarps) {
        uint4* o = reinterpret_cast<uint4*>(out + (int64_t)t * h);
        if (dropped[t]) {
            for (int v = lane; v < h / 8; v += 32) o[v] = make_uint4(0, 0, 0, 0);
            if (dlogits) for (int e = lane; e < E; e += 32) dlogits[(int64_t)t * E + e] = 0.0f;
            continue;
        }
        uint32_t mask = 0;
        int ex[8];
        float dl[8];
        for (int j = 0; j < k; ++j) {
            ex[j] = experts_loc[(int64_t)t * k + j];
            mask |= 1u << (ex[j] / el);
        }
        const bool router = wr != nullptr;
        if (router) {
            float g[8], dg[8];
            for (int j = 0; j < k; ++j) {
                g[j] = gates[(int64_t)t * k + j];
                dg[j] = dgates[(int64_t)t * k + j];
            }
            softmax_topk_bwd(g, dg, k, dl);
            if (dlogits) {
                for (int e = lane; e < E; e += 32) {
                    float v = 0.0f;
                    for (int j = 0; j < k; ++j) v = (ex[j] == e) ? dl[j] : v;
                    dlogits[(int64_t)t * E + e] = v;
                }
            }
        }
        for (int v = lane; v < nv16; v += 32) {
            float acc[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] = 0.0f;
            for (int r = 0; r < n; ++r) {
                if (!(mask >> r & 1u)) continue;
                const uint4* sp = reinterpret_cast<const uint4*>(stage + ((int64_t)t * n + r) * h);
                const uint4 s0 = sp[2 * v], s1 = sp[2 * v + 1];
                const uint32_t w[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float2 p = unpack_bf16x2(w[q]);
                    acc[2 * q] += p.x;
                    acc[2 * q + 1] += p.y;
                }
            }
            if (router) {
                for (int j = 0; j < k; ++j) {
                    const uint4* wp = reinterpret_cast<const uint4*>(wr + (int64_t)ex[j] * h);
                    const uint4 w0 = wp[2 * v], w1 = wp[2 * v + 1];
                    const uint32_t w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float2 p = unpack_bf16x2(w[q]);
                        acc[2 * q] += dl[j] * p.x;
                        acc[2 * q + 1] += dl[j] * p.y;
                    }
                }
            }
            o[2 * v] = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                                  pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
            o[2 * v + 1] = make_uint4(pack_bf16x2(acc[8], acc[9]), pack_bf16x2(acc[10], acc[11]),
                                      pack_bf16x2(acc[12], acc[13]), pack_bf16x2(acc[14], acc[15]));
        }
    }
}

// dgate of each permuted row = sum over f-tiles of the epilogue partials
// (fixed order, deterministic), scattered to (source rank, t_local*k+slot).
static __global__ void dgate_reduce_kernel(const float* __restrict__ part, int n_parts,
                                    const int32_t* __restrict__ row_dst, const int32_t* nrows_pad,
                                    float* const* __restrict__ dst_bufs) {
    // one warp per row: coalesced reads of the row's partials, fixed-order
    // lane sums then a butterfly (deterministic)
    const int total = *nrows_pad;
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int pp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; pp < total; pp += nw) {
        const int d = row_dst[pp];
        if (d < 0) continue;
        float s = 0.0f;
        for (int q = lane; q < n_parts; q += 32) s += part[(int64_t)pp * n_parts + q];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) dst_bufs[d >> 27][d & ((1 << 27) - 1)] = s;
    }
}

// Router weight gradient dwr[e, c] = sum_t dlogits[t, e] * x[t, c] (fp32).
// Pass 1: block (column tile of 256, token chunk of 128) -> partial [chunk][E][h];
// pass 2: fixed-order sum over chunks (deterministic). E <= 32 per pass.
constexpr int kRwChunk = 128;
template <int EB>
static __global__ void router_wgrad_partial_kernel(const float* __restrict__ dlogits, const uint16_t* __restrict__ x,
                                            int T, int h, int E, float* __restrict__ part) {
    __shared__ float s_dl[kRwChunk * EB];
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int t0 = blockIdx.y * kRwChunk;
    const int nt = min(kRwChunk, T - t0);
    for (int e0 = 0; e0 < E; e0 += EB) {
        const int ne = min(EB, E - e0);
        __syncthreads();
        for (int i = threadIdx.x; i < nt * EB; i += blockDim.x) {
            const int tt = i / EB, ee = i % EB;
            s_dl[i] = ee < ne ? dlogits[(int64_t)(t0 + tt) * E + e0 + ee] : 0.0f;
        }
        __syncthreads();
        float acc[EB];
#pragma unroll
        for (int q = 0; q < EB; ++q) acc[q] = 0.0f;
        if (c < h) {
            for (int tt = 0; tt < nt; ++tt) {
                const float xv = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(x)[(int64_t)(t0 + tt) * h + c]);
#pragma unroll
                for (int q = 0; q < EB; ++q) acc[q] = fmaf(s_dl[tt * EB + q], xv, acc[q]);
            }
#pragma unroll
            for (int q = 0; q < EB; ++q)
                if (q < ne) part[((int64_t)blockIdx.y * E + e0 + q) * h + c] = acc[q];
        }
    }
}

// E <= 8: 8 columns per thread (one 16 B load of x per token, the chunk's 32
// tokens' loads in flight), token chunks of kRw8Chunk; same [chunk][E][h]
// partial layout, summed in fixed chunk order by router_wgrad_reduce_kernel.
constexpr int kRw8Chunk = 32;
static __global__ void __launch_bounds__(128) router_wgrad_partial8_kernel(
    const float* __restrict__ dlogits, const uint16_t* __restrict__ x, int T, int h, int E,
    float* __restrict__ part) {
    __shared__ float s_dl[kRw8Chunk * 8];
    const int c0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
    const int t0 = blockIdx.y * kRw8Chunk;
    const int nt = min(kRw8Chunk, T - t0);
    for (int i = threadIdx.x; i < kRw8Chunk * 8; i += blockDim.x) {
        const int tt = i >> 3, ee = i & 7;
        s_dl[i] = (tt < nt && ee < E) ? dlogits[(int64_t)(t0 + tt) * E + ee] : 0.0f;
    }
    __syncthreads();
    if (c0 >= h) return;
    float acc[8][8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[q][j] = 0.0f;
    const uint4* xp = reinterpret_cast<const uint4*>(x + (int64_t)t0 * h + c0);
    const int hv = h / 8;
#pragma unroll 1
    for (int tt = 0; tt < kRw8Chunk; tt += 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = tt + u < nt ? __ldg(xp + (int64_t)(tt + u) * hv) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float2 a = unpack_bf16x2(v[u].x), b = unpack_bf16x2(v[u].y), c = unpack_bf16x2(v[u].z),
                         d = unpack_bf16x2(v[u].w);
            const float xf[8] = {a.x, a.y, b.x, b.y, c.x, c.y, d.x, d.y};
            const float* dl = s_dl + (tt + u) * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float g = dl[q];
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[q][j] = fmaf(g, xf[j], acc[q][j]);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        if (q < E) {
            float4* o = reinterpret_cast<float4*>(part + ((int64_t)blockIdx.y * E + q) * h + c0);
            o[0] = make_float4(acc[q][0], acc[q][1], acc[q][2], acc[q][3]);
            o[1] = make_float4(acc[q][4], acc[q][5], acc[q][6], acc[q][7]);
        }
    }
}

static __global__ void router_wgrad_reduce_kernel(const float* __restrict__ part, int nchunks, int E, int h,
                                           float* __restrict__ dwr) {
    const int64_t n = (int64_t)E * h;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float s = 0.0f;
        for (int q = 0; q < nchunks; ++q) s += part[(int64_t)q * n + i];
        dwr[i] = s;
    }
}

// Same sum for many chunks (n % 4 == 0): a 256-thread block owns 32 float4
// outputs; its 8 warps take every 8th chunk (8 loads in flight each) and the
// 8 partial sums are added in warp order through shared memory (fixed order,
// deterministic).
static __global__ void __launch_bounds__(256) chunk_sum4_kernel(const float* __restrict__ part, int nchunks,
                                                                 int64_t n, float* __restrict__ out) {
    __shared__ float4 s_p[8][32];
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int64_t n4 = n / 4;
    const int64_t i = (int64_t)blockIdx.x * 32 + lane;
    const float4* p4 = reinterpret_cast<const float4*>(part);
    float4 s = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (i < n4) {
        for (int q0 = g; q0 < nchunks; q0 += 64) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int q = q0 + 8 * u;
                v[u] = q < nchunks ? p4[(int64_t)q * n4 + i] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) { s.x += v[u].x; s.y += v[u].y; s.z += v[u].z; s.w += v[u].w; }
        }
    }
    s_p[g][lane] = s;
    __syncthreads();
    if (g == 0 && i < n4) {
        float4 t = s_p[0][lane];
#pragma unroll
        for (int w = 1; w < 8; ++w) { t.x += s_p[w][lane].x; t.y += s_p[w][lane].y; t.z += s_p[w][lane].z; t.w += s_p[w][lane].w; }
        reinterpret_cast<float4*>(out)[i] = t;
    }
}

// Pack w1 [el][2f][h] ([a | b] rows) into the interleaved layout the fused
// SwiGLU epilogue expects: per 128-row block, 64 a-rows then 64 b-rows.
static __global__ void pack_w1_kernel(const uint16_t* __restrict__ w1, uint16_t* __restrict__ w1p, int el,
                               int f, int h) {
    const int64_t rows = (int64_t)el * 2 * f;
    const int nvec = h / 8;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const int e = (int)(r / (2 * f));
        const int j = (int)(r % (2 * f));
        const int blk = j >> 7, w = j & 127;   // [a 64 | b 64] per 128-row block
        const int src_j = w < 64 ? blk * 64 + w : f + blk * 64 + (w - 64);
        const uint4* s = reinterpret_cast<const uint4*>(w1 + ((int64_t)e * 2 * f + src_j) * h);
        uint4* d = reinterpret_cast<uint4*>(w1p + r * h);
        for (int v = threadIdx.x; v < nvec; v += blockDim.x) d[v] = s[v];
    }
}

// Copy this rank's routing (experts/gates for its T_r tokens) into every
// rank's global routing table at offset rank*T_r*k.
static __global__ void publish_meta_kernel(const int32_t* __restrict__ ex, const float* __restrict__ gt,
                                    int count, int offset, int32_t* const* ex_bufs,
                                    float* const* gt_bufs, int n) {
    for (int p = 0; p < n; ++p)
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
            ex_bufs[p][offset + i] = ex[i];
            gt_bufs[p][offset + i] = gt[i];
        }
}

// Device-side barrier over NVLink: rank r stores `epoch` into slot[r] of
// every peer's flag array (release, system scope), then waits until its own
// array holds >= epoch for all peers. The epoch lives in device memory and
// is bumped on the device (bump = 1 at the first barrier of a pass), so the
// whole layer can be captured once in a CUDA graph and replayed. Bounded
// spin -> *err = 1 on timeout instead of a hang.
// `stamp` (optional): %globaltimer at entry and at release, so the wait for the
// slowest rank (rank-imbalance idle) is measured inside graph-replayed steps.
static __global__ void flag_barrier_kernel(uint32_t* const* peer_flags, int slot, int n, int rank,
                                    uint32_t* epoch_dev, int bump, unsigned long long timeout_ns,
                                    int* err, unsigned long long* stamp = nullptr, int debug = 0) {
    __shared__ uint32_t s_epoch;
    if (threadIdx.x == 0) {
        if (stamp) stamp[0] = globaltimer();
        uint32_t e = *epoch_dev;
        if (bump) *epoch_dev = ++e;
        s_epoch = e;
    }
    __syncthreads();
    const uint32_t epoch = s_epoch;
    const int i = threadIdx.x;
    if (i < n) {
        __threadfence_system();
        st_release_sys(peer_flags[i] + slot * 64 + rank, epoch);
    }
    __syncthreads();
    if (i < n) {
        const uint32_t* mine = peer_flags[rank] + slot * 64 + i;
        const uint64_t t0 = globaltimer();
        while ((int32_t)(ld_acquire_sys(mine) - epoch) < 0) {
            if (globaltimer() - t0 > timeout_ns) {
                atomicExch(err, 1);
                break;
            }
        }
    }
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[1] = globaltimer();
    // debug mode (err != nullptr and debug): after the release every peer's flag of
    // this slot must hold exactly this epoch — older means the wait was broken,
    // newer means a peer ran ahead into the next use of the slot
    if (debug && i < n) {
        const uint32_t v = ld_acquire_sys(peer_flags[rank] + slot * 64 + i);
        if (v != epoch) atomicExch(err, 16 + slot);
    }
}

// Debug-mode check of the fused-dispatch protocol after a fused GEMM: every
// 128-row block of the permuted operand received exactly 128 arrivals (each
// padded row claimed and landed once), no block past the end received any,
// the row-claim counter passed the end, deduplicated rows landed exactly once,
// and (ag_rs) every all-gather chunk of every peer landed completely.
static __global__ void dispatch_check_kernel(const uint32_t* __restrict__ ready, int nblocks_alloc,
                                             const int32_t* nrows_pad, const int* row_claim, int ag_rows,
                                             const uint32_t* __restrict__ row_done, const int32_t* __restrict__ pad_tok,
                                             const uint32_t* __restrict__ ag_ready, int n, int self, int tokens_per_rank,
                                             int* err) {
    const int total = *nrows_pad;
    const int nb = total / 128;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nblocks_alloc; b += gridDim.x * blockDim.x)
        if (ready[b] != (b < nb ? 128u : 0u)) atomicExch(err, 8);
    if (blockIdx.x == 0 && threadIdx.x == 0 && *row_claim < ag_rows + total) atomicExch(err, 9);
    if (row_done)
        for (int pp = blockIdx.x * blockDim.x + threadIdx.x; pp < total; pp += gridDim.x * blockDim.x)
            if (pad_tok[pp] >= 0 && row_done[pp] != 1u) atomicExch(err, 10);
    if (ag_ready) {
        const int nch = (tokens_per_rank + 63) / 64;
        for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n * nch; c += gridDim.x * blockDim.x) {
            const int src = c / nch, ch = c - src * nch;
            const uint32_t want = src == self ? 0u : (uint32_t)min(64, tokens_per_rank - ch * 64);
            if (ag_ready[c] != want) atomicExch(err, 11);
        }
    }
}

// %globaltimer stamp at a phase boundary (trace of graph-replayed steps)
static __global__ void stamp_kernel(unsigned long long* p) {
    if (threadIdx.x == 0) *p = globaltimer();
}

// K1 fast path: router weights staged in shared memory as fp32 (E*h*4 bytes),
// one warp per FOUR tokens so every shared-memory weight load feeds four
// FMAs; x streamed with 16-byte loads, RD vectors per token in flight per lane
// (a rolling prefetch ring, 8 KB per warp) and the first ones issued before
// the weights are staged, so the kernel runs at the x stream's HBM rate.
// E is processed in groups of 8.
static __global__ void __launch_bounds__(256, 1) router_logits_smem_kernel(
    const uint16_t* __restrict__ x, const uint16_t* __restrict__ wr, int T, int h, int E,
    float* __restrict__ logits) {
    extern __shared__ __align__(16) float s_wf[];  // [E][h] fp32
    constexpr int RD = 4;                           // prefetch depth (iterations of 32 vectors)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int nvec = h / 8;
    auto ldx = [&](int t0, int nt, int i, int v) -> uint4 {
        return (i < nt && v < nvec) ? __ldg(reinterpret_cast<const uint4*>(x + (int64_t)(t0 + i) * h) + v)
                                    : make_uint4(0, 0, 0, 0);
    };
    int t0 = (blockIdx.x * wpb + warp) * 4;
    uint4 xn[RD][4];
    {   // the first task's first vectors fly while W_r is staged
        const int nt = t0 < T ? min(4, T - t0) : 0;
#pragma unroll
        for (int d = 0; d < RD; ++d)
#pragma unroll
            for (int i = 0; i < 4; ++i) xn[d][i] = ldx(t0, nt, i, lane + 32 * d);
    }
    {   // W_r -> smem fp32 with 8 independent 16 B loads in flight per thread
        const int nw = E * h / 8;
        constexpr int WU = 8;
        for (int i0 = threadIdx.x; i0 < nw; i0 += blockDim.x * WU) {
            uint4 v[WU];
#pragma unroll
            for (int u = 0; u < WU; ++u)
                if (i0 + u * (int)blockDim.x < nw) v[u] = __ldg(reinterpret_cast<const uint4*>(wr) + i0 + u * blockDim.x);
#pragma unroll
            for (int u = 0; u < WU; ++u) {
                const int i = i0 + u * blockDim.x;
                if (i < nw) {
                    const float2 a = unpack_bf16x2(v[u].x), b = unpack_bf16x2(v[u].y),
                                 c = unpack_bf16x2(v[u].z), d = unpack_bf16x2(v[u].w);
                    reinterpret_cast<float4*>(s_wf)[2 * i] = make_float4(a.x, a.y, b.x, b.y);
                    reinterpret_cast<float4*>(s_wf)[2 * i + 1] = make_float4(c.x, c.y, d.x, d.y);
                }
            }
        }
    }
    __syncthreads();
    bool primed = true;
    for (; t0 < T; t0 += gridDim.x * wpb * 4) {
        const int nt = min(4, T - t0);
        for (int e0 = 0; e0 < E; e0 += 8) {
            if (!primed) {
#pragma unroll
                for (int d = 0; d < RD; ++d)
#pragma unroll
                    for (int i = 0; i < 4; ++i) xn[d][i] = ldx(t0, nt, i, lane + 32 * d);
            }
            primed = false;
            float acc[4][8];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 8; ++q) acc[i][q] = 0.0f;
            for (int v0 = lane; v0 < nvec; v0 += 32 * RD) {
#pragma unroll
                for (int d = 0; d < RD; ++d) {
                    const int v = v0 + 32 * d;
                    float xf[4][8];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint4 xv = xn[d][i];
                        const float2 a = unpack_bf16x2(xv.x), b = unpack_bf16x2(xv.y),
                                     c = unpack_bf16x2(xv.z), dd = unpack_bf16x2(xv.w);
                        xf[i][0] = a.x; xf[i][1] = a.y; xf[i][2] = b.x; xf[i][3] = b.y;
                        xf[i][4] = c.x; xf[i][5] = c.y; xf[i][6] = dd.x; xf[i][7] = dd.y;
                        xn[d][i] = ldx(t0, nt, i, v + 32 * RD);   // refill the slot RD steps ahead
                    }
                    if (v < nvec) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            if (e0 + q < E) {
                                const float4 w0 = reinterpret_cast<const float4*>(s_wf + (int64_t)(e0 + q) * h)[2 * v];
                                const float4 w1 = reinterpret_cast<const float4*>(s_wf + (int64_t)(e0 + q) * h)[2 * v + 1];
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    float s = acc[i][q];
                                    s = fmaf(xf[i][0], w0.x, s); s = fmaf(xf[i][1], w0.y, s);
                                    s = fmaf(xf[i][2], w0.z, s); s = fmaf(xf[i][3], w0.w, s);
                                    s = fmaf(xf[i][4], w1.x, s); s = fmaf(xf[i][5], w1.y, s);
                                    s = fmaf(xf[i][6], w1.z, s); s = fmaf(xf[i][7], w1.w, s);
                                    acc[i][q] = s;
                                }
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float a = acc[i][q];
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
                    if (lane == 0 && i < nt && e0 + q < E) logits[(int64_t)(t0 + i) * E + e0 + q] = a;
                }
        }
    }
}

// K1 for E <= 8 (Mixtral shape): logits[T, E] = x . W_r^T with warp-level
// bf16 tensor-core MMAs (m16n8k16, fp32 accumulate; n = 8 = E). A CTA owns 16
// tokens; its 8 warps split h into 8 slices and the slices' partial logits
// are summed in fixed warp order through shared memory (deterministic). The
// contraction index inside every 32-column window is permuted identically for
// x and W_r (lane c's fragment slots {2c, 2c+1, 2c+8, 2c+9} of step t are the
// physical columns 8c + 4t + {0..3}), so each lane feeds two MMAs from one
// 16-byte load per token row: the kernel is a pure stream of x.
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// nsplit > 1: the h columns of a 16-token block are split over nsplit CTAs
// (4096 tokens -> 256 x nsplit CTAs: several per SM, so HBM sees enough
// requests in flight); each writes its fp32 partial sums to part[] and the
// last CTA to arrive (counter cnt[block], reset by it) adds the partials in
// split order — deterministic whatever the arrival order — then runs the
// top-k + softmax.
static __global__ void __launch_bounds__(256) router_logits_mma_kernel(
    const uint16_t* __restrict__ x, const uint16_t* __restrict__ wr, int T, int h, int E,
    float* __restrict__ logits, int k, int32_t* __restrict__ experts, float* __restrict__ gates,
    int nsplit = 1, float* __restrict__ part = nullptr, unsigned* __restrict__ cnt = nullptr) {
    __shared__ float red[8][16][8];
    __shared__ float s_lg[16][8];
    __shared__ int s_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, c = lane & 3;
    const int blk = blockIdx.x / nsplit, sp = blockIdx.x - blk * nsplit;
    const int t0 = blk * 16;
    const int slice = h / (8 * nsplit), k_lo = sp * (h / nsplit) + warp * slice;
    const bool r0 = t0 + g < T, r1 = t0 + g + 8 < T, ev = g < E;
    const uint4* xa = reinterpret_cast<const uint4*>(x + (int64_t)(t0 + g) * h + k_lo) + c;
    const uint4* xb = reinterpret_cast<const uint4*>(x + (int64_t)(t0 + g + 8) * h + k_lo) + c;
    const uint4* wb = reinterpret_cast<const uint4*>(wr + (int64_t)g * h + k_lo) + c;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    constexpr int WB = 4;   // 32-column windows per batch; two batches in flight (24 x 16 B per lane)
    const uint4 z = make_uint4(0, 0, 0, 0);
    const int nwin = slice / 32;
    auto load = [&](uint4 (&va)[WB], uint4 (&vb)[WB], uint4 (&vw)[WB], int w0) {
#pragma unroll
        for (int u = 0; u < WB; ++u) {
            const bool in = w0 + u < nwin;
            va[u] = (in && r0) ? __ldg(xa + (w0 + u) * 4) : z;
            vb[u] = (in && r1) ? __ldg(xb + (w0 + u) * 4) : z;
            vw[u] = (in && ev) ? __ldg(wb + (w0 + u) * 4) : z;
        }
    };
    auto mma = [&](const uint4 (&va)[WB], const uint4 (&vb)[WB], const uint4 (&vw)[WB]) {
#pragma unroll
        for (int u = 0; u < WB; ++u) {
            mma_bf16_16816(acc, va[u].x, vb[u].x, va[u].y, vb[u].y, vw[u].x, vw[u].y);
            mma_bf16_16816(acc, va[u].z, vb[u].z, va[u].w, vb[u].w, vw[u].z, vw[u].w);
        }
    };
    uint4 a0[WB], b0[WB], w0v[WB], a1[WB], b1[WB], w1v[WB];
    load(a0, b0, w0v, 0);
    for (int w0 = 0; w0 < nwin; w0 += 2 * WB) {
        load(a1, b1, w1v, w0 + WB);         // next batch in flight during this one's MMAs
        mma(a0, b0, w0v);
        if (w0 + 2 * WB < nwin) load(a0, b0, w0v, w0 + 2 * WB);
        if (w0 + WB < nwin) mma(a1, b1, w1v);
    }
    red[warp][g][2 * c] = acc[0];
    red[warp][g][2 * c + 1] = acc[1];
    red[warp][g + 8][2 * c] = acc[2];
    red[warp][g + 8][2 * c + 1] = acc[3];
    __syncthreads();
    if (threadIdx.x < 128) {
        const int r = threadIdx.x >> 3, e = threadIdx.x & 7;
        float sum = red[0][r][e];
#pragma unroll
        for (int w = 1; w < 8; ++w) sum += red[w][r][e];
        if (nsplit == 1) {
            s_lg[r][e] = sum;
            if (e < E && t0 + r < T) logits[(int64_t)(t0 + r) * E + e] = sum;
        } else {
            part[((int64_t)blk * nsplit + sp) * 128 + threadIdx.x] = sum;
            __threadfence();
        }
    }
    if (nsplit > 1) {
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(&cnt[blk], 1u) == (unsigned)(nsplit - 1);
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        if (threadIdx.x < 128) {
            const int r = threadIdx.x >> 3, e = threadIdx.x & 7;
            float sum = __ldcg(part + (int64_t)blk * nsplit * 128 + threadIdx.x);
            for (int q = 1; q < nsplit; ++q) sum += __ldcg(part + ((int64_t)blk * nsplit + q) * 128 + threadIdx.x);
            s_lg[r][e] = sum;
            if (e < E && t0 + r < T) logits[(int64_t)(t0 + r) * E + e] = sum;
        }
        if (threadIdx.x == 0) cnt[blk] = 0u;   // ready for the next call (graph replays)
    }
    __syncthreads();
    // top-k + softmax of the CTA's 16 tokens, two per warp (the separate
    // topk_from_logits launch folded in)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int r = 2 * warp + q;
        if (t0 + r < T)
            topk_select(s_lg[r], E, k, experts + (int64_t)(t0 + r) * k, gates + (int64_t)(t0 + r) * k, lane);
    }
}

// ffn_norm (graph.cpp:267): y = x * rsqrt(mean(x^2) + eps) * gamma, one warp
// per token, rstd kept for the backward (the reference remats the norm in
// backward, graph.cpp:355-359; here it is recomputed from x and rstd).
static __global__ void rmsnorm_fwd_kernel(const uint16_t* __restrict__ x, const float* __restrict__ gamma,
                                          float eps, int T, int h, uint16_t* __restrict__ y,
                                          float* __restrict__ rstd) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int t = warp; t < T; t += nw) {
        const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)t * h);
        float ss = 0.0f;
        for (int v = lane; v < h / 8; v += 32) {
            const uint4 a = xr[v];
            const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 p = unpack_bf16x2(w[q]);
                ss += p.x * p.x + p.y * p.y;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
        const float r = rsqrtf(ss / (float)h + eps);
        if (lane == 0) rstd[t] = r;
        uint4* yr = reinterpret_cast<uint4*>(y + (int64_t)t * h);
        for (int v = lane; v < h / 8; v += 32) {
            const uint4 a = xr[v];
            const float4 g0 = reinterpret_cast<const float4*>(gamma)[2 * v];
            const float4 g1 = reinterpret_cast<const float4*>(gamma)[2 * v + 1];
            const float2 p0 = unpack_bf16x2(a.x), p1 = unpack_bf16x2(a.y), p2 = unpack_bf16x2(a.z), p3 = unpack_bf16x2(a.w);
            yr[v] = make_uint4(pack_bf16x2(p0.x * r * g0.x, p0.y * r * g0.y), pack_bf16x2(p1.x * r * g0.z, p1.y * r * g0.w),
                               pack_bf16x2(p2.x * r * g1.x, p2.y * r * g1.y), pack_bf16x2(p3.x * r * g1.z, p3.y * r * g1.w));
        }
    }
}

// RMSNorm backward: dx = rstd * (gamma*g - xhat * mean(xhat*gamma*g)), xhat = x*rstd
static __global__ void rmsnorm_bwd_kernel(const uint16_t* __restrict__ x, const float* __restrict__ gamma,
                                          const float* __restrict__ rstd, const uint16_t* __restrict__ g,
                                          int T, int h, uint16_t* __restrict__ dx) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int t = warp; t < T; t += nw) {
        const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)t * h);
        const uint4* gr = reinterpret_cast<const uint4*>(g + (int64_t)t * h);
        const float r = rstd[t];
        float dot = 0.0f;
        for (int v = lane; v < h / 8; v += 32) {
            const uint4 a = xr[v], b = gr[v];
            const float4 g0 = reinterpret_cast<const float4*>(gamma)[2 * v];
            const float4 g1 = reinterpret_cast<const float4*>(gamma)[2 * v + 1];
            const float gm[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
            const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 px = unpack_bf16x2(wa[q]), pg = unpack_bf16x2(wb[q]);
                dot += px.x * r * gm[2 * q] * pg.x + px.y * r * gm[2 * q + 1] * pg.y;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
        const float mean = dot / (float)h;
        uint4* dr = reinterpret_cast<uint4*>(dx + (int64_t)t * h);
        for (int v = lane; v < h / 8; v += 32) {
            const uint4 a = xr[v], b = gr[v];
            const float4 g0 = reinterpret_cast<const float4*>(gamma)[2 * v];
            const float4 g1 = reinterpret_cast<const float4*>(gamma)[2 * v + 1];
            const float gm[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
            const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
            uint32_t o[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 px = unpack_bf16x2(wa[q]), pg = unpack_bf16x2(wb[q]);
                o[q] = pack_bf16x2(r * (gm[2 * q] * pg.x - px.x * r * mean),
                                   r * (gm[2 * q + 1] * pg.y - px.y * r * mean));
            }
            dr[v] = make_uint4(o[0], o[1], o[2], o[3]);
        }
    }
}

// d gamma partials: part[chunk, c] = sum over the chunk's tokens of g * xhat
static __global__ void rmsnorm_dgamma_partial_kernel(const uint16_t* __restrict__ x, const float* __restrict__ rstd,
                                                     const uint16_t* __restrict__ g, int T, int h,
                                                     float* __restrict__ part) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int t0 = blockIdx.y * kRwChunk, t1 = min(T, t0 + kRwChunk);
    if (c >= h) return;
    float acc = 0.0f;
    for (int t = t0; t < t1; ++t) {
        const float xv = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(x)[(int64_t)t * h + c]);
        const float gv = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(g)[(int64_t)t * h + c]);
        acc += gv * xv * rstd[t];
    }
    part[(int64_t)blockIdx.y * h + c] = acc;
}

static __global__ void f32_to_bf16_kernel(const float* __restrict__ in, uint16_t* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const __nv_bfloat16 b = __float2bfloat16_rn(in[i]);
        out[i] = *reinterpret_cast<const uint16_t*>(&b);
    }
}

static __global__ void source_rank_kernel(int32_t* src, int T, int tokens_per_rank) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x)
        src[t] = t / tokens_per_rank;
}

}  // namespace moe
