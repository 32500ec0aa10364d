// f32path.cu — the fp32 MoE layer forward (BASELINE configs[0]: 4096
// tokens, hidden 1024, ffn 2816, 8 experts top-2, fp32, checked against the
// fp32 CPU oracle at 1e-5). Same operator chain as the bf16 path
// (router -> capacity drop -> permutation -> dispatch -> fc1 -> SwiGLU (->
// gate) -> fc2 -> gather -> combine, graph.cpp:254-311).
//
// Expert GEMMs on the tcgen05 tensor cores with fp32 accuracy ("bf16x6"): every
// fp32 operand x is split exactly into three bf16 pieces hi = bf16(x),
// mid = bf16(x - hi), lo = bf16(x - hi - mid) (|x - hi - mid - lo| <= 2^-24 |x|).
// With A' = [A_hi, A_hi, A_mid, A_hi, A_lo, A_mid] and B' = [B_hi, B_mid, B_hi,
// B_lo, B_hi, B_mid] along K, A'.B'^T holds every cross term down to 2^-16
// (hi.hi, hi.mid, mid.hi, hi.lo, lo.hi, mid.mid; the dropped ones are <= 2^-24)
// and bf16 products are exact. Measured (scripts/probe_accum.py): the tcgen05
// fp32 accumulator truncates at every MMA (all-positive data: -1.4e-5 relative
// bias at K = 4096, -8.2e-5 at 16384, linear in K), so the error grows with the
// number of MMAs adding into one accumulator. The hi.hi part (contraction K)
// and the 2^-8-smaller corrections (5K) therefore run as two GEMMs over column
// windows of the same split operands, summed in fp32 by the next kernel: the
// truncation error stays that of a K-long accumulation (~1e-6 at these shapes)
// instead of a 6K-long one (5.4e-5 measured in one pass). 6 bf16 MMAs cost what
// 3 tf32 MMAs would. MOE_F32_FFMA=1 selects the FFMA grouped GEMMs, for A/B.
#include <cmath>

#include <cstdlib>

#include "common.cuh"
#include "gemm.h"
#include "layer_kernels.cuh"
#include "runtime.h"

namespace moe {
namespace {

constexpr int FT_M = 128, FT_N = 128, FT_K = 8;

// C[Mrows, N] (+ row scatter) = A[Mrows, K] . B_g[N, K]^T, grouped by padded
// row segments (multiples of 128). EPI 0: store rows; 1: scatter rows to
// dst_row (+ optional row gate) for the combine.
template <int EPI>
__global__ void __launch_bounds__(256) ffma_grouped_gemm_kernel(
    const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C, int N, int K,
    int G, const int32_t* __restrict__ gpad_off, const int32_t* __restrict__ row_dst,
    const float* __restrict__ row_gate, int64_t ldc) {
    __shared__ float As[2][FT_K][FT_M];
    __shared__ float Bs[2][FT_K][FT_N];
    const int row0 = blockIdx.x * FT_M;
    const int n0 = blockIdx.y * FT_N;
    if (row0 >= gpad_off[G]) return;
    int lo = 0, hi = G - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (gpad_off[mid] <= row0) lo = mid;
        else hi = mid - 1;
    }
    const float* Bg = B + (int64_t)lo * N * K;
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;  // 16 x 16 threads, 8 x 8 outputs each
    // loader mapping: 128 rows x 8 k = 1024 floats per operand = 4 per thread
    const int lr = tid / 2, lk = (tid % 2) * 4;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
    const float* ap = A + (int64_t)(row0 + lr) * K + lk;
    const bool bvalid = n0 + lr < N;
    const float* bp = Bg + (int64_t)(n0 + lr) * K + lk;
    float4 ra = *reinterpret_cast<const float4*>(ap);
    float4 rb = bvalid ? *reinterpret_cast<const float4*>(bp) : make_float4(0, 0, 0, 0);
    int buf = 0;
    for (int k0 = 0; k0 < K; k0 += FT_K) {
        As[buf][lk + 0][lr] = ra.x; As[buf][lk + 1][lr] = ra.y; As[buf][lk + 2][lr] = ra.z; As[buf][lk + 3][lr] = ra.w;
        Bs[buf][lk + 0][lr] = rb.x; Bs[buf][lk + 1][lr] = rb.y; Bs[buf][lk + 2][lr] = rb.z; Bs[buf][lk + 3][lr] = rb.w;
        __syncthreads();
        if (k0 + FT_K < K) {
            ra = *reinterpret_cast<const float4*>(ap + k0 + FT_K);
            rb = bvalid ? *reinterpret_cast<const float4*>(bp + k0 + FT_K) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int kk = 0; kk < FT_K; ++kk) {
            float a[8], b[8];
            *reinterpret_cast<float4*>(&a[0]) = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
            *reinterpret_cast<float4*>(&a[4]) = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
            *reinterpret_cast<float4*>(&b[0]) = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
            *reinterpret_cast<float4*>(&b[4]) = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        buf ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = row0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        float* dst;
        float gsc = 1.0f;
        if (EPI == 0) {
            dst = C + (int64_t)r * ldc;
        } else {
            const int d = row_dst[r];
            if (d < 0) continue;
            dst = C + (int64_t)(d & ((1 << 27) - 1)) * ldc;
            if (row_gate) gsc = row_gate[r];
        }
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            const int c = n0 + h2 * 64 + tx * 4;
            if (c < N) {
                float4 v = make_float4(acc[i][h2 * 4] * gsc, acc[i][h2 * 4 + 1] * gsc, acc[i][h2 * 4 + 2] * gsc,
                                       acc[i][h2 * 4 + 3] * gsc);
                *reinterpret_cast<float4*>(dst + c) = v;
            }
        }
    }
}

// fc2_in[r, j] = a * silu(b) (* gate) with fc1 = [a | b] (numerics.cpp:262-268)
__global__ void swiglu_f32_kernel(const float* __restrict__ fc1, const float* __restrict__ row_gate,
                                  const int32_t* nrows, int f, float* __restrict__ out) {
    const int64_t n = (int64_t)(*nrows) * f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / f, j = i - r * f;
        const float a = fc1[r * 2 * f + j], b = fc1[r * 2 * f + f + j];
        float v = a * (b / (1.0f + expf(-b)));
        if (row_gate) v *= row_gate[r];
        out[i] = v;
    }
}

__global__ void combine_f32_kernel(const float* __restrict__ stage, const uint8_t* __restrict__ dropped,
                                   int T, int k, int h, float* __restrict__ y) {
    const int64_t n = (int64_t)T * h;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / h, c = i - t * h;
        float acc = 0.0f;
        if (!(dropped && dropped[t]))
            for (int j = 0; j < k; ++j) acc += stage[(t * k + j) * h + c];
        y[i] = acc;
    }
}

__global__ void router_f32_kernel(const float* __restrict__ x, const float* __restrict__ wr, int T, int h,
                                  int E, float* __restrict__ logits) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int64_t p = warp; p < (int64_t)T * E; p += nw) {
        const int64_t t = p / E, e = p - t * E;
        float acc = 0.0f;
        for (int c = lane; c < h; c += 32) acc = fmaf(x[t * h + c], wr[e * h + c], acc);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) logits[p] = acc;
    }
}

// ---- bf16x6 operand preparation ----
struct Bf3 { uint16_t hi, mid, lo; };
__device__ __forceinline__ uint16_t bf16_bits(float v) {
    __nv_bfloat16 b = __float2bfloat16_rn(v);
    return *reinterpret_cast<uint16_t*>(&b);
}
__device__ __forceinline__ float bf16_val(uint16_t u) { return __uint_as_float((uint32_t)u << 16); }
__device__ __forceinline__ Bf3 split3(float x) {
    Bf3 r;
    r.hi = bf16_bits(x);
    const float r1 = x - bf16_val(r.hi);     // exact
    r.mid = bf16_bits(r1);
    const float r2 = r1 - bf16_val(r.mid);   // exact
    r.lo = bf16_bits(r2);
    return r;
}
// piece order along K: A side [hi, hi, mid, hi, lo, mid], B side [hi, mid, hi, lo, hi, mid].
// 8 consecutive elements per thread: one 16-byte store per piece.
__device__ __forceinline__ void store6x8(uint16_t* d, int64_t K, const float (&v)[8], int b_side) {
    uint32_t hi[4], mid[4], lo[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const Bf3 a = split3(v[2 * q]), b = split3(v[2 * q + 1]);
        hi[q] = (uint32_t)a.hi | ((uint32_t)b.hi << 16);
        mid[q] = (uint32_t)a.mid | ((uint32_t)b.mid << 16);
        lo[q] = (uint32_t)a.lo | ((uint32_t)b.lo << 16);
    }
    const uint4 H = make_uint4(hi[0], hi[1], hi[2], hi[3]), M = make_uint4(mid[0], mid[1], mid[2], mid[3]),
                Lo = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    const uint4 seq_a[6] = {H, H, M, H, Lo, M}, seq_b[6] = {H, M, H, Lo, H, M};
#pragma unroll
    for (int j = 0; j < 6; ++j) *reinterpret_cast<uint4*>(d + j * K) = b_side ? seq_b[j] : seq_a[j];
}
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
// dst row r [6K] (bf16) = the pieces of src row r [K] (fp32); K % 8 == 0
__global__ void split6_rows_kernel(const float* __restrict__ src, int64_t rows, int K, int b_side,
                                   uint16_t* __restrict__ dst) {
    const int kv = K / 8;
    const int64_t n = rows * kv;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / kv;
        const int c = (int)(i - r * kv) * 8;
        float v[8];
        load8(src + r * K + c, v);
        store6x8(dst + r * 6 * K + c, K, v, b_side);
    }
}
// dispatch + split: padded row pp = pieces of x[token of pp] (A side), zeros for pads
__global__ void gather_split6_kernel(const int32_t* __restrict__ pad_row_tok, const int32_t* nrows_pad, int k,
                                     const float* __restrict__ x, int h, uint16_t* __restrict__ dst) {
    const int hv = h / 8;
    const int64_t n = (int64_t)(*nrows_pad) * hv;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pp = i / hv;
        const int c = (int)(i - pp * hv) * 8;
        const int tk = pad_row_tok[pp];
        float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (tk >= 0) load8(x + (int64_t)(tk / k) * h + c, v);
        store6x8(dst + pp * 6 * h + c, h, v, 0);
    }
}
// SwiGLU (+ gate) of fc1 rows (main + correction GEMM outputs), written as fc2 A-side pieces
__global__ void swiglu_split6_kernel(const float* __restrict__ fc1, const float* __restrict__ fc1c,
                                     const float* __restrict__ row_gate, const int32_t* nrows, int f,
                                     uint16_t* __restrict__ dst) {
    const int fv = f / 8;
    const int64_t n = (int64_t)(*nrows) * fv;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / fv;
        const int j = (int)(i - r * fv) * 8;
        float a[8], ac[8], b[8], bc[8], v[8];
        load8(fc1 + r * 2 * f + j, a);
        load8(fc1c + r * 2 * f + j, ac);
        load8(fc1 + r * 2 * f + f + j, b);
        load8(fc1c + r * 2 * f + f + j, bc);
        const float g = row_gate ? row_gate[r] : 1.0f;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float av = a[q] + ac[q], bv = b[q] + bc[q];
            v[q] = av * (bv / (1.0f + expf(-bv))) * g;
        }
        store6x8(dst + r * 6 * f + j, f, v, 0);
    }
}
// y[t] = sum over slots (fixed order) of the expert output rows of (t, slot)
__global__ void combine_rows_f32_kernel(const float* __restrict__ rows, const float* __restrict__ rows_c,
                                        const int32_t* __restrict__ inv, int T, int k, int h, float* __restrict__ y) {
    const int64_t n = (int64_t)T * h;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / h, c = i - t * h;
        float acc = 0.0f;
        for (int j = 0; j < k; ++j) {
            const int pp = inv[t * k + j];
            if (pp >= 0) acc += rows[(int64_t)pp * h + c] + rows_c[(int64_t)pp * h + c];
        }
        y[i] = acc;
    }
}

__global__ void iota_src_kernel(int32_t* src, int T) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) src[t] = 0;
}

template <class T>
moe_status salloc(T** p, size_t n, cudaStream_t s) {
    MOE_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T), s));
    return MOE_OK;
}

}  // namespace
}  // namespace moe

using namespace moe;

extern "C" moe_status moe_ffn_forward_f32(const float* d_x, const float* d_w1, const float* d_w2,
                                          const float* d_wr, int64_t T, int64_t h, int64_t f, int64_t E,
                                          int64_t k, double capacity_factor, int32_t gate_order,
                                          const int32_t* d_experts_in, const float* d_gates_in,
                                          float* d_y, int32_t* d_experts, float* d_gates,
                                          float* d_logits, uint8_t* d_dropped, moe_stream_t stream) {
    MOE_CHECK_ARG(d_x && d_w1 && d_w2 && d_y && d_experts && d_gates && d_dropped, "null argument");
    MOE_CHECK_ARG(T >= 1 && h % 8 == 0 && f % 4 == 0 && E >= 1 && k >= 1 && k <= 8 && k <= E,
                  "need h % 8 == 0, f % 4 == 0, 1 <= k <= min(8, E)");
    MOE_CHECK_ARG(d_experts_in || d_wr, "need a router weight or injected routing");
    cudaStream_t s = (cudaStream_t)stream;
    {
        // the per-call work buffers come from the device's stream-ordered pool;
        // keep freed blocks in the pool (default threshold 0 returns them to the
        // driver at every synchronisation, and re-mapping ~2 GB per call costs
        // more than the layer itself)
        int dev = 0;
        cudaGetDevice(&dev);
        static uint64_t pool_done = 0;
        if (!(pool_done >> (dev & 63) & 1)) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            pool_done |= 1ull << (dev & 63);
        }
    }
    const int64_t Mp = T * k + E * 128;
    float *logits = d_logits, *x_perm = nullptr, *fc1 = nullptr, *fc2_in = nullptr, *stage = nullptr,
          *row_gate = nullptr;
    int32_t *src = nullptr, *rmi = nullptr, *cnt = nullptr, *oe = nullptr, *osr = nullptr, *offs = nullptr,
            *rows = nullptr, *gpr = nullptr, *gpo = nullptr, *ptok = nullptr, *rdst = nullptr;
    void* ws = nullptr;
    bool own_logits = false;
    if (!d_experts_in && !logits) {
        MOE_TRY(salloc(&logits, T * E, s));
        own_logits = true;
    }
    MOE_TRY(salloc(&src, T, s));
    MOE_TRY(salloc(&rmi, T * k, s));
    MOE_TRY(salloc(&cnt, E, s));
    MOE_TRY(salloc(&oe, T * k, s));
    MOE_TRY(salloc(&osr, T * k, s));
    MOE_TRY(salloc(&offs, E + 1, s));
    MOE_TRY(salloc(&rows, 1, s));
    MOE_TRY(salloc(&gpr, E, s));
    MOE_TRY(salloc(&gpo, E + 1, s));
    MOE_TRY(salloc(&ptok, Mp, s));
    MOE_TRY(salloc(&rdst, Mp, s));
    MOE_TRY(salloc(&row_gate, Mp, s));
    MOE_TRY(salloc(&x_perm, Mp * h, s));
    MOE_TRY(salloc(&fc1, Mp * 2 * f, s));
    MOE_TRY(salloc(&fc2_in, Mp * f, s));
    MOE_TRY(salloc(&stage, T * k * h, s));
    MOE_TRY(salloc(reinterpret_cast<uint8_t**>(&ws), permute_workspace_bytes(T, E, k, 1), s));
    // router (fp32) or injected routing
    if (d_experts_in) {
        MOE_CUDA_TRY(cudaMemcpyAsync(d_experts, d_experts_in, T * k * 4, cudaMemcpyDeviceToDevice, s));
        MOE_CUDA_TRY(cudaMemcpyAsync(d_gates, d_gates_in, T * k * 4, cudaMemcpyDeviceToDevice, s));
    } else {
        router_f32_kernel<<<kNumSMs * 8, 256, 0, s>>>(d_x, d_wr, (int)T, (int)h, (int)E, logits);
        count_launch();
        MOE_TRY(launch_topk_from_logits(logits, T, E, k, d_experts, d_gates, s));
    }
    if (capacity_factor > 0.0)
        MOE_TRY(launch_capacity_drop(d_experts, T, E, k, 1, capacity_factor, d_dropped, s));
    else
        MOE_CUDA_TRY(cudaMemsetAsync(d_dropped, 0, T, s));
    iota_src_kernel<<<64, 256, 0, s>>>(src, (int)T);
    count_launch();
    MOE_TRY(launch_permute(d_experts, src, d_dropped, T, E, k, 1, 0, 1, rmi, cnt, oe, osr, offs, rows, ws,
                           gpr, gpo, ptok, 128, s));
    row_info_kernel<<<(unsigned)E, 256, 0, s>>>(gpo, gpr, offs, ptok, d_gates, (int)k, (int)T, row_gate, rdst);
    count_launch();
    const bool gate_after_ = gate_order == MOE_GATE_AFTER_FC2;
    static const bool ffma = getenv("MOE_F32_FFMA") != nullptr;
    if (!ffma && h % 64 == 0 && f % 64 == 0) {
        // ---- bf16x6 tensor-core path ----
        const int cg = double(T * k) / double(E) >= 256.0 ? 2 : 1;
        uint16_t *xs = nullptr, *w1s = nullptr, *w2s = nullptr, *f2s = nullptr;
        float* orow = nullptr;
        int32_t* inv = nullptr;
        MOE_TRY(salloc(&xs, Mp * 6 * h, s));
        MOE_TRY(salloc(&w1s, E * 2 * f * 6 * h, s));
        MOE_TRY(salloc(&w2s, E * h * 6 * f, s));
        MOE_TRY(salloc(&f2s, Mp * 6 * f, s));
        MOE_TRY(salloc(&orow, Mp * h, s));
        MOE_TRY(salloc(&inv, T * k, s));
        const int grid = kNumSMs * 8;
        split6_rows_kernel<<<grid, 256, 0, s>>>(d_w1, E * 2 * f, (int)h, 1, w1s);
        split6_rows_kernel<<<grid, 256, 0, s>>>(d_w2, E * h, (int)f, 1, w2s);
        gather_split6_kernel<<<grid, 256, 0, s>>>(ptok, gpo + E, (int)k, d_x, (int)h, xs);
        count_launch(3);
        // two GEMMs over column windows of the split operands (row stride 6K):
        // main = hi.hi (K columns), corr = the five correction blocks (5K columns)
        auto window = [](CUtensorMap* m, const uint16_t* base, int64_t rows, int64_t Kp, int64_t first,
                         int64_t width, int box_rows) {
            return make_tmap_2d(m, base + first, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (uint64_t)width,
                                (uint64_t)rows, (uint64_t)(6 * Kp * 2), 64, (uint32_t)box_rows);
        };
        float* fc1c = nullptr;
        float* orowc = nullptr;
        MOE_TRY(salloc(&fc1c, Mp * 2 * f, s));
        MOE_TRY(salloc(&orowc, Mp * h, s));
        for (int part = 0; part < 2; ++part) {
            const int64_t first = part ? h : 0, width = part ? 5 * h : h;
            GemmPlan p1;
            p1.cg = cg;
            p1.epi = EPI_STORE_F32;
            MOE_TRY(window(&p1.ta, xs, Mp, h, first, width, 128));
            MOE_TRY(window(&p1.tb, w1s, E * 2 * f, h, first, width, 256 / cg));
            GemmArgs a1{};
            a1.G = (int)E;
            a1.group_rows = gpr;
            a1.N = (int)(2 * f);
            a1.K = (int)width;
            a1.b_group_stride = (int)(2 * f);
            a1.out = part ? fc1c : fc1;
            a1.ldo = 2 * f;
            MOE_TRY(gemm_launch(p1, a1, s));
        }
        swiglu_split6_kernel<<<grid, 256, 0, s>>>(fc1, fc1c, gate_after_ ? nullptr : row_gate, gpo + E, (int)f, f2s);
        count_launch();
        for (int part = 0; part < 2; ++part) {
            const int64_t first = part ? f : 0, width = part ? 5 * f : f;
            GemmPlan p2;
            p2.cg = cg;
            p2.epi = EPI_STORE_F32;
            MOE_TRY(window(&p2.ta, f2s, Mp, f, first, width, 128));
            MOE_TRY(window(&p2.tb, w2s, E * h, f, first, width, 256 / cg));
            GemmArgs a2{};
            a2.G = (int)E;
            a2.group_rows = gpr;
            a2.N = (int)h;
            a2.K = (int)width;
            a2.b_group_stride = (int)h;
            a2.out = part ? orowc : orow;
            a2.ldo = h;
            a2.row_gate = row_gate;
            a2.gate_rows = gate_after_ ? 1 : 0;
            MOE_TRY(gemm_launch(p2, a2, s));
        }
        MOE_CUDA_TRY(cudaMemsetAsync(inv, 0xff, T * k * 4, s));
        inverse_rows_kernel<<<kNumSMs * 2, 256, 0, s>>>(ptok, gpo + E, inv);
        combine_rows_f32_kernel<<<grid, 256, 0, s>>>(orow, orowc, inv, (int)T, (int)k, (int)h, d_y);
        count_launch(2);
        MOE_CUDA_TRY(cudaGetLastError());
        void* bufs[] = {src, rmi, cnt, oe, osr, offs, rows, gpr, gpo, ptok, rdst, row_gate, x_perm, fc1, fc2_in,
                        stage, ws, xs, w1s, w2s, f2s, orow, inv, fc1c, orowc};
        for (void* b : bufs) cudaFreeAsync(b, s);
        if (own_logits) cudaFreeAsync(logits, s);
        return MOE_OK;
    }
    // dispatch: fp32 rows copied as 2x bf16-width rows (16-byte vector copy)
    const uint16_t* srcbuf = reinterpret_cast<const uint16_t*>(d_x);
    const uint16_t** tab = nullptr;
    MOE_TRY(salloc(&tab, 1, s));
    MOE_CUDA_TRY(cudaMemcpyAsync(tab, &srcbuf, sizeof(void*), cudaMemcpyHostToDevice, s));
    dispatch_rows_kernel<<<kNumSMs * 4, 256, 0, s>>>(ptok, gpo + E, (int)k, (int)T, (int)(2 * h), tab,
                                                     reinterpret_cast<uint16_t*>(x_perm));
    count_launch();
    const bool gate_after = gate_order == MOE_GATE_AFTER_FC2;
    const dim3 g1((unsigned)(Mp / FT_M), (unsigned)((2 * f + FT_N - 1) / FT_N));
    ffma_grouped_gemm_kernel<0><<<g1, 256, 0, s>>>(x_perm, d_w1, fc1, (int)(2 * f), (int)h, (int)E, gpo,
                                                    nullptr, nullptr, 2 * f);
    swiglu_f32_kernel<<<kNumSMs * 8, 256, 0, s>>>(fc1, gate_after ? nullptr : row_gate, gpo + E, (int)f, fc2_in);
    const dim3 g2((unsigned)(Mp / FT_M), (unsigned)((h + FT_N - 1) / FT_N));
    ffma_grouped_gemm_kernel<1><<<g2, 256, 0, s>>>(fc2_in, d_w2, stage, (int)h, (int)f, (int)E, gpo, rdst,
                                                    gate_after ? row_gate : nullptr, h);
    combine_f32_kernel<<<kNumSMs * 8, 256, 0, s>>>(stage, d_dropped, (int)T, (int)k, (int)h, d_y);
    count_launch(4);
    MOE_CUDA_TRY(cudaGetLastError());
    void* bufs[] = {src, rmi, cnt, oe, osr, offs, rows, gpr, gpo, ptok, rdst, row_gate, x_perm, fc1, fc2_in,
                    stage, ws, tab};
    for (void* b : bufs) cudaFreeAsync(b, s);
    if (own_logits) cudaFreeAsync(logits, s);
    return MOE_OK;
}
