// routing.cu — K1 router/top-k and K2 routing maps (capacity drop, stable
// permutation, tile layout, balance counts) for sm_100a.
//
// Bit-exact contracts (integer): /root/reference/proj/core/src/routing.cpp
//   capacity drop            :113-131
//   build_scatter_map        :135-187
//   sort_tokens_for_tiles    :189-217
//   balance_metrics (counts) :219-262
#include <cmath>

#include "common.cuh"
#include "topk.cuh"
#include "runtime.h"

namespace moe {

// ---------------------------------------------------------------------------
// K1: router logits + top-k + softmax over the selected logits
// ---------------------------------------------------------------------------
// One warp per token. Each lane accumulates partial dot products for a chunk
// of up to 32 experts over its slice of h (16-byte vectors), then a warp
// butterfly reduction. Wr rows are read through L1/L2 (E*h*2 bytes, reused
// by every token of the block).
__global__ void router_topk_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ wr,
                                   int T, int h, int E, int k, float* __restrict__ logits,
                                   int32_t* __restrict__ experts, float* __restrict__ gates) {
    extern __shared__ float s_logits[];  // [warps][E]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    float* lg = s_logits + warp * E;
    for (int t = blockIdx.x * wpb + warp; t < T; t += gridDim.x * wpb) {
        const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)t * h);
        for (int e0 = 0; e0 < E; e0 += 8) {
            const int ne = min(8, E - e0);
            float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int v = lane; v < h / 8; v += 32) {
                const uint4 xv = __ldg(xr + v);
                const float2 x0 = unpack_bf16x2(xv.x), x1 = unpack_bf16x2(xv.y),
                             x2 = unpack_bf16x2(xv.z), x3 = unpack_bf16x2(xv.w);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (q < ne) {
                        const uint4 wv = __ldg(reinterpret_cast<const uint4*>(wr + (int64_t)(e0 + q) * h) + v);
                        const float2 w0 = unpack_bf16x2(wv.x), w1 = unpack_bf16x2(wv.y),
                                     w2 = unpack_bf16x2(wv.z), w3 = unpack_bf16x2(wv.w);
                        float a = acc[q];
                        a = fmaf(x0.x, w0.x, a); a = fmaf(x0.y, w0.y, a);
                        a = fmaf(x1.x, w1.x, a); a = fmaf(x1.y, w1.y, a);
                        a = fmaf(x2.x, w2.x, a); a = fmaf(x2.y, w2.y, a);
                        a = fmaf(x3.x, w3.x, a); a = fmaf(x3.y, w3.y, a);
                        acc[q] = a;
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                float a = acc[q];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
                if (lane == 0 && q < ne) lg[e0 + q] = a;
            }
        }
        __syncwarp();
        if (logits)
            for (int e = lane; e < E; e += 32) logits[(int64_t)t * E + e] = lg[e];
        topk_select(lg, E, k, experts + (int64_t)t * k, gates + (int64_t)t * k, lane);
        __syncwarp();
    }
}

__global__ void topk_from_logits_kernel(const float* __restrict__ logits, int T, int E, int k,
                                        int32_t* __restrict__ experts, float* __restrict__ gates) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    for (int t = blockIdx.x * wpb + warp; t < T; t += gridDim.x * wpb)
        topk_select(logits + (int64_t)t * E, E, k, experts + (int64_t)t * k,
                    gates + (int64_t)t * k, lane);
}

// ---------------------------------------------------------------------------
// capacity drop (routing.cpp:113-131)
// ---------------------------------------------------------------------------
// One CTA. Loads per group via a block histogram; fast path when no group is
// over capacity. Otherwise warp 0 scans 32-token chunks from the top: a token
// can only be dropped if one of its groups is over capacity at the start of
// its chunk (loads only decrease), so only ballot candidates are resolved
// serially, in descending token order. Group loads live in lane g (n <= 32).
__global__ void capacity_drop_kernel(const int32_t* __restrict__ experts, int T, int k,
                                     int per, int n_groups, long long capacity,
                                     uint8_t* __restrict__ dropped) {
    __shared__ unsigned long long s_load[32];
    __shared__ int s_any_over;
    for (int i = threadIdx.x; i < 32; i += blockDim.x) s_load[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < T * k; i += blockDim.x)
        atomicAdd(&s_load[experts[i] / per], 1ull);
    for (int t = threadIdx.x; t < T; t += blockDim.x) dropped[t] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        int any = 0;
        for (int g = 0; g < n_groups; ++g) any |= (long long)s_load[g] > capacity;
        s_any_over = any;
    }
    __syncthreads();
    if (!s_any_over || threadIdx.x >= 32) return;

    const int lane = threadIdx.x;
    long long load = lane < n_groups ? (long long)s_load[lane] : 0;
    for (int base = T - 1; base >= 0; base -= 32) {
        // early exit once no group is over capacity
        if (__ballot_sync(0xffffffffu, load > capacity) == 0) break;
        const int t = base - lane;  // lane 0 = highest token of the chunk
        unsigned gmask = 0;
        if (t >= 0)
            for (int j = 0; j < k; ++j) gmask |= 1u << (experts[(int64_t)t * k + j] / per);
        const unsigned overmask = __ballot_sync(0xffffffffu, load > capacity);
        unsigned cand = __ballot_sync(0xffffffffu, t >= 0 && (gmask & overmask) != 0);
        while (cand) {
            const int src = __ffs(cand) - 1;
            cand &= cand - 1;
            const int tt = base - src;
            const unsigned m = __shfl_sync(0xffffffffu, gmask, src);
            const unsigned over_now = __ballot_sync(0xffffffffu, load > capacity);
            if (m & over_now) {
                // drop whole token: decrement every group once per slot
                int cnt = 0;
                if (lane < n_groups && ((m >> lane) & 1))
                    for (int j = 0; j < k; ++j) cnt += (experts[(int64_t)tt * k + j] / per) == lane;
                load -= cnt;
                if (lane == 0) dropped[tt] = 1;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K2: stable counting-sort permutation (build_scatter_map)
// ---------------------------------------------------------------------------
// Entries i = t*k + slot are processed in index order. Bin of a local entry =
// (expert - first) * n_src + source_rank; the reference's order
// (expert, source_rank, token) is exactly (bin, i) because within a token
// the k experts are distinct. Three passes:
//   1. per-chunk bin histograms (+ global per-expert counts)
//   2. one CTA scans (bin-major, chunk-minor) -> chunk offsets; expert offsets
//   3. per-chunk stable scatter: warp match_any ranks + cross-warp prefix
constexpr int kPermThreads = 256;
// entries per chunk (multiple of kPermThreads): small problems use 256 so that
// the histogram / scatter passes spread over more CTAs (Mixtral N=1: 8 -> 32)
static int perm_chunk(int64_t n_ent) { return n_ent <= 65536 ? 256 : 1024; }

__global__ void permute_hist_kernel(const int32_t* __restrict__ experts,
                                    const int32_t* __restrict__ src,
                                    const uint8_t* __restrict__ dropped, int T, int k, int E,
                                    int first, int el, int n_src, int* __restrict__ chunk_cnt,
                                    int* __restrict__ per_expert_counts, int chunk) {
    extern __shared__ int s_h[];  // [nbins] then [E]
    const int nbins = el * n_src;
    int* s_e = s_h + nbins;
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) s_h[b] = 0;
    for (int e = threadIdx.x; e < E; e += blockDim.x) s_e[e] = 0;
    __syncthreads();
    const int64_t n_ent = (int64_t)T * k;
    const int64_t beg = (int64_t)blockIdx.x * chunk;
    for (int64_t i = beg + threadIdx.x; i < beg + chunk && i < n_ent; i += blockDim.x) {
        const int t = (int)(i / k);
        if (dropped && dropped[t]) continue;
        const int e = experts[i];
        atomicAdd(&s_e[e], 1);
        if (e >= first && e < first + el) atomicAdd(&s_h[(e - first) * n_src + src[t]], 1);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nbins; b += blockDim.x)
        chunk_cnt[(int64_t)blockIdx.x * nbins + b] = s_h[b];
    for (int e = threadIdx.x; e < E; e += blockDim.x)
        if (s_e[e]) atomicAdd(&per_expert_counts[e], s_e[e]);
}

// Exclusive scan of a[0..n) in shared memory by the whole (1024-thread) block:
// up to 4 consecutive items per thread, warp shuffles, then a scan of the 32
// warp totals. Returns the total (to every thread).
__device__ int block_exclusive_scan(int* a, int n, int* s_warp) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (n + blockDim.x - 1) / blockDim.x;   // items per thread (<= 4 used here)
    const int beg = tid * per;
    int loc[4] = {0, 0, 0, 0};
    int sum = 0;
    for (int q = 0; q < per && q < 4; ++q) {
        loc[q] = beg + q < n ? a[beg + q] : 0;
        sum += loc[q];
    }
    int incl = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += u;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
        int wi = w;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, wi, off);
            if (lane >= off) wi += u;
        }
        s_warp[lane] = wi - w;           // exclusive warp offsets
        if (lane == 31) s_warp[32] = wi;  // block total
    }
    __syncthreads();
    int run = s_warp[warp] + incl - sum;
    for (int q = 0; q < per && q < 4; ++q) {
        if (beg + q < n) a[beg + q] = run;
        run += loc[q];
    }
    const int total = s_warp[32];
    __syncthreads();
    return total;
}

// One CTA (1024 threads): column prefix per bin over chunks (8 chunk loads in
// flight per thread), block scans over bins and over the padded expert sizes.
// Same results as a serial scan (integer sums).
__global__ void permute_scan_kernel(int* __restrict__ chunk_cnt, int nchunks, int nbins, int el,
                                    int n_src, int* __restrict__ expert_offsets,
                                    int* __restrict__ rows_out, int* __restrict__ group_pad_rows,
                                    int* __restrict__ group_pad_off, int pad) {
    extern __shared__ int s_tot[];  // [nbins + 1] then [el + 1] padded sizes
    __shared__ int s_warp[33];
    int* s_pad = s_tot + nbins + 1;
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
        int acc = 0;
        int c = 0;
        for (; c + 8 <= nchunks; c += 8) {
            int v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = chunk_cnt[(int64_t)(c + u) * nbins + b];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                chunk_cnt[(int64_t)(c + u) * nbins + b] = acc;  // exclusive within bin
                acc += v[u];
            }
        }
        for (; c < nchunks; ++c) {
            const int v = chunk_cnt[(int64_t)c * nbins + b];
            chunk_cnt[(int64_t)c * nbins + b] = acc;
            acc += v;
        }
        s_tot[b] = acc;
    }
    __syncthreads();
    const int total = block_exclusive_scan(s_tot, nbins, s_warp);
    if (threadIdx.x == 0) {
        s_tot[nbins] = total;
        *rows_out = total;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < el; e += blockDim.x) {
        const int beg = s_tot[e * n_src];
        const int end = s_tot[(e + 1) * n_src];
        expert_offsets[e] = beg;
        s_pad[e] = (end - beg + pad - 1) / pad * pad;
    }
    if (threadIdx.x == 0) expert_offsets[el] = total;
    __syncthreads();
    if (group_pad_rows) {
        for (int e = threadIdx.x; e < el; e += blockDim.x) group_pad_rows[e] = s_pad[e];
        __syncthreads();
        const int ptotal = block_exclusive_scan(s_pad, el, s_warp);
        for (int e = threadIdx.x; e < el; e += blockDim.x) group_pad_off[e] = s_pad[e];
        if (threadIdx.x == 0) group_pad_off[el] = ptotal;
    }
    // add bin base to every chunk's exclusive offsets
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
        const int base = s_tot[b];
        for (int c = 0; c < nchunks; ++c) chunk_cnt[(int64_t)c * nbins + b] += base;
    }
}

struct PermuteOut {
    int32_t* row_map_in;
    int32_t* out_expert;
    int32_t* out_source_rank;
    // padded-space outputs for the GEMM path (may be null)
    const int32_t* expert_offsets;
    const int32_t* group_pad_off;
    int32_t* pad_row_tok;  // [Mp] t*k+slot, -1 for pad rows (filled elsewhere)
};

__global__ void permute_scatter_kernel(const int32_t* __restrict__ experts,
                                       const int32_t* __restrict__ src,
                                       const uint8_t* __restrict__ dropped, int T, int k,
                                       int first, int el, int n_src,
                                       const int* __restrict__ chunk_off, PermuteOut out, int chunk) {
    extern __shared__ int s_w[];  // [8 warps][nbins] then running[nbins]
    const int nbins = el * n_src;
    int* s_run = s_w + 8 * nbins;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
        s_run[b] = chunk_off[(int64_t)blockIdx.x * nbins + b];
        for (int w = 0; w < 8; ++w) s_w[w * nbins + b] = 0;
    }
    __syncthreads();
    const int64_t n_ent = (int64_t)T * k;
    const int64_t beg = (int64_t)blockIdx.x * chunk;
    for (int round = 0; round < chunk / kPermThreads; ++round) {
        const int64_t i = beg + round * kPermThreads + threadIdx.x;
        int bin = -1, e = -1, t = 0;
        if (i < n_ent) {
            t = (int)(i / k);
            if (!(dropped && dropped[t])) {
                e = experts[i];
                if (e >= first && e < first + el) bin = (e - first) * n_src + src[t];
            }
        }
        const unsigned peers = __match_any_sync(0xffffffffu, bin);
        const int rank_w = __popc(peers & ((1u << lane) - 1));
        if (bin >= 0 && rank_w == 0) s_w[warp * nbins + bin] = __popc(peers);
        __syncthreads();
        if (bin >= 0) {
            int off = s_run[bin] + rank_w;
            for (int w = 0; w < warp; ++w) off += s_w[w * nbins + bin];
            out.row_map_in[off] = (int32_t)i;
            out.out_expert[off] = e;
            out.out_source_rank[off] = src[t];
            if (out.pad_row_tok) {
                const int g = e - first;
                out.pad_row_tok[off - out.expert_offsets[g] + out.group_pad_off[g]] = (int32_t)i;
            }
        }
        __syncthreads();
        for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
            int s = 0;
            for (int w = 0; w < 8; ++w) {
                s += s_w[w * nbins + b];
                s_w[w * nbins + b] = 0;
            }
            s_run[b] += s;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// tile layout (sort_tokens_for_tiles) — one thread per tile
// ---------------------------------------------------------------------------
__global__ void tile_layout_kernel(const int32_t* __restrict__ out_src,
                                   const int32_t* __restrict__ expert_offsets, int el, int first,
                                   int tile_rows, int32_t* __restrict__ t_expert,
                                   int32_t* __restrict__ t_begin, int32_t* __restrict__ t_end,
                                   uint64_t* __restrict__ t_mask, int32_t* __restrict__ n_tiles) {
    __shared__ int s_pref[1025];
    // el <= 1024 local experts
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int e = 0; e < el; ++e) {
            s_pref[e] = acc;
            const int c = expert_offsets[e + 1] - expert_offsets[e];
            acc += (c + tile_rows - 1) / tile_rows;
        }
        s_pref[el] = acc;
        *n_tiles = acc;
    }
    __syncthreads();
    const int total = s_pref[el];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        int lo = 0, hi = el - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_pref[mid] <= i) lo = mid;
            else hi = mid - 1;
        }
        const int e = lo;
        const int b = expert_offsets[e] + (i - s_pref[e]) * tile_rows;
        const int end = min(b + tile_rows, expert_offsets[e + 1]);
        uint64_t m = 0;
        for (int r = b; r < end; ++r) m |= 1ull << out_src[r];
        t_expert[i] = first + e;
        t_begin[i] = b;
        t_end[i] = end;
        t_mask[i] = m;
    }
}

// ---------------------------------------------------------------------------
// balance counts (routing.cpp:219-262, integer part)
// ---------------------------------------------------------------------------
__global__ void balance_counts_kernel(const int32_t* __restrict__ experts,
                                      const uint8_t* __restrict__ dropped, int T, int k, int per,
                                      int n, int64_t* load, int64_t* assigned, int64_t* ndrop) {
    __shared__ unsigned long long s_l[64], s_a[64], s_d;
    for (int i = threadIdx.x; i < 64; i += blockDim.x) s_l[i] = s_a[i] = 0;
    if (threadIdx.x == 0) s_d = 0;
    __syncthreads();
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
        const bool d = dropped && dropped[t];
        if (d) atomicAdd(&s_d, 1ull);
        for (int j = 0; j < k; ++j) {
            const int g = experts[(int64_t)t * k + j] / per;
            atomicAdd(&s_a[g], 1ull);
            if (!d) atomicAdd(&s_l[g], 1ull);
        }
    }
    __syncthreads();
    for (int g = threadIdx.x; g < n; g += blockDim.x) {
        if (s_l[g]) atomicAdd(reinterpret_cast<unsigned long long*>(&load[g]), s_l[g]);
        if (s_a[g]) atomicAdd(reinterpret_cast<unsigned long long*>(&assigned[g]), s_a[g]);
    }
    if (threadIdx.x == 0 && s_d) atomicAdd(reinterpret_cast<unsigned long long*>(ndrop), s_d);
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
moe_status launch_router_topk(const uint16_t* x, const uint16_t* wr, int64_t T, int64_t h,
                              int64_t E, int64_t k, float* logits, int32_t* experts, float* gates,
                              cudaStream_t s) {
    MOE_CHECK_ARG(T >= 0 && h > 0 && h % 8 == 0, "router: h must be a positive multiple of 8");
    MOE_CHECK_ARG(E >= 1 && E <= 1024 && k >= 1 && k <= 8 && k <= E, "router: need 1<=k<=min(8,E), E<=1024");
    if (T == 0) return MOE_OK;
    const int threads = 256, wpb = threads / 32;
    const size_t smem = (size_t)wpb * E * sizeof(float);
    int grid = (int)std::min<int64_t>((T + wpb - 1) / wpb, kNumSMs * 8);
    if (smem > 48 * 1024)
        MOE_CUDA_TRY(cudaFuncSetAttribute(router_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    router_topk_kernel<<<grid, threads, smem, s>>>(x, wr, (int)T, (int)h, (int)E, (int)k, logits,
                                                   experts, gates);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

moe_status launch_topk_from_logits(const float* logits, int64_t T, int64_t E, int64_t k,
                                   int32_t* experts, float* gates, cudaStream_t s) {
    MOE_CHECK_ARG(E >= 1 && k >= 1 && k <= 8 && k <= E, "topk: need 1<=k<=min(8,E)");
    if (T == 0) return MOE_OK;
    int grid = (int)std::min<int64_t>((T + 7) / 8, kNumSMs * 8);
    topk_from_logits_kernel<<<grid, 256, 0, s>>>(logits, (int)T, (int)E, (int)k, experts, gates);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

moe_status launch_capacity_drop(const int32_t* experts, int64_t T, int64_t E, int64_t k,
                                int64_t n_groups, double cf, uint8_t* dropped, cudaStream_t s) {
    MOE_CHECK_ARG(T >= 0, "tokens must be >= 0");
    MOE_CHECK_ARG(E >= 1 && k >= 1, "counts must be >= 1");
    MOE_CHECK_ARG(k <= E, "top_k must not exceed num_experts");
    MOE_CHECK_ARG(n_groups >= 1, "n_groups must be >= 1");
    MOE_CHECK_ARG(E % n_groups == 0, "num_experts must divide evenly across groups");
    MOE_CHECK_ARG(cf > 0.0, "capacity_factor must be > 0");
    MOE_CHECK_ARG(n_groups <= 32, "capacity drop on device supports n_groups <= 32");
    if (T == 0) return MOE_OK;
    // routing.cpp:115-117, evaluated in double exactly as the reference does
    const long long capacity = static_cast<long long>(
        std::ceil(cf * static_cast<double>(T) * static_cast<double>(k) / static_cast<double>(n_groups)));
    capacity_drop_kernel<<<1, 1024, 0, s>>>(experts, (int)T, (int)k, (int)(E / n_groups),
                                           (int)n_groups, capacity, dropped);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

size_t permute_workspace_bytes(int64_t T, int64_t E, int64_t k, int64_t n_src) {
    const int64_t nchunks = (T * k + perm_chunk(T * k) - 1) / perm_chunk(T * k);
    return (size_t)std::max<int64_t>(nchunks, 1) * (size_t)(E * n_src) * sizeof(int) + 256;
}

moe_status launch_permute(const int32_t* experts, const int32_t* src, const uint8_t* dropped,
                          int64_t T, int64_t E, int64_t k, int64_t n, int64_t my_rank,
                          int64_t n_src, int32_t* row_map_in, int32_t* per_expert_counts,
                          int32_t* out_expert, int32_t* out_src, int32_t* expert_offsets,
                          int32_t* rows, void* workspace, int32_t* group_pad_rows,
                          int32_t* group_pad_off, int32_t* pad_row_tok, int pad,
                          cudaStream_t s) {
    MOE_CHECK_ARG(n >= 1, "n must be >= 1");
    MOE_CHECK_ARG(my_rank >= 0 && my_rank < n, "my_rank out of range");
    MOE_CHECK_ARG(E % n == 0, "num_experts must be divisible by n");
    MOE_CHECK_ARG(n_src >= 1 && n_src <= 64, "source ranks must lie in [0, 64)");
    const int el = (int)(E / n);
    const int first = (int)(my_rank * el);
    const int nbins = el * (int)n_src;
    MOE_CHECK_ARG(nbins <= 4096, "permute supports (E/n)*n_src <= 4096 bins");
    const int64_t n_ent = T * k;
    const int chunk = perm_chunk(n_ent);
    const int nchunks = (int)std::max<int64_t>((n_ent + chunk - 1) / chunk, 1);
    int* chunk_cnt = static_cast<int*>(workspace);
    MOE_CUDA_TRY(cudaMemsetAsync(per_expert_counts, 0, sizeof(int32_t) * E, s));
    const size_t sm1 = sizeof(int) * (nbins + E);
    if (sm1 > 48 * 1024)
        MOE_CUDA_TRY(cudaFuncSetAttribute(permute_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1));
    permute_hist_kernel<<<nchunks, kPermThreads, sm1, s>>>(experts, src, dropped, (int)T, (int)k,
                                                           (int)E, first, el, (int)n_src,
                                                           chunk_cnt, per_expert_counts, chunk);
    count_launch();
    const size_t sm2 = sizeof(int) * (nbins + 1 + el + 1);
    permute_scan_kernel<<<1, 1024, sm2, s>>>(chunk_cnt, nchunks, nbins, el, (int)n_src,
                                             expert_offsets, rows, group_pad_rows, group_pad_off,
                                             pad);
    count_launch();
    PermuteOut po{row_map_in, out_expert, out_src, expert_offsets, group_pad_off, pad_row_tok};
    const size_t sm3 = sizeof(int) * 9 * nbins;
    if (sm3 > 48 * 1024)
        MOE_CUDA_TRY(cudaFuncSetAttribute(permute_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3));
    permute_scatter_kernel<<<nchunks, kPermThreads, sm3, s>>>(experts, src, dropped, (int)T,
                                                              (int)k, first, el, (int)n_src,
                                                              chunk_cnt, po, chunk);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

moe_status launch_tile_layout(const int32_t* out_src, const int32_t* expert_offsets, int64_t el,
                              int64_t first, int64_t tile_rows, int32_t* t_expert,
                              int32_t* t_begin, int32_t* t_end, uint64_t* t_mask,
                              int32_t* n_tiles, cudaStream_t s) {
    MOE_CHECK_ARG(tile_rows >= 1, "tile_rows must be >= 1");
    MOE_CHECK_ARG(el >= 1 && el <= 1024, "local experts must be in [1, 1024]");
    tile_layout_kernel<<<kNumSMs, 256, 0, s>>>(out_src, expert_offsets, (int)el, (int)first,
                                               (int)tile_rows, t_expert, t_begin, t_end, t_mask,
                                               n_tiles);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

moe_status launch_balance_counts(const int32_t* experts, const uint8_t* dropped, int64_t T,
                                 int64_t E, int64_t k, int64_t n, int64_t* load,
                                 int64_t* assigned, int64_t* ndrop, cudaStream_t s) {
    MOE_CHECK_ARG(n >= 1 && n <= 64, "n must be in [1, 64]");
    MOE_CHECK_ARG(E % n == 0, "incompatible group count");
    MOE_CUDA_TRY(cudaMemsetAsync(load, 0, sizeof(int64_t) * n, s));
    MOE_CUDA_TRY(cudaMemsetAsync(assigned, 0, sizeof(int64_t) * n, s));
    MOE_CUDA_TRY(cudaMemsetAsync(ndrop, 0, sizeof(int64_t), s));
    if (T == 0) return MOE_OK;
    const int grid = (int)std::min<int64_t>((T + 255) / 256, kNumSMs);
    balance_counts_kernel<<<grid, 256, 0, s>>>(experts, dropped, (int)T, (int)k, (int)(E / n),
                                               (int)n, load, assigned, ndrop);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

}  // namespace moe
