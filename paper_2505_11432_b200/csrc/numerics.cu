// numerics.cu — the reference's low-precision numerics on the GPU, bit-exact
// (binary64 arithmetic in the same operation order):
//   round_to        numerics.cpp:50-68  (RNE to bf16 / e4m3 / fp32; e4m3
//                                         saturates at 448, bf16 overflows to inf)
//   quantize        numerics.cpp:88-160 (block absmax -> scale -> codes; four
//                                         granularities)
//   emulate_reduce  numerics.cpp:172-192 (ring_bf16 vs a2a_fp32 combine order)
// These back the FP8 communication option and the combine-reduction semantics
// of the data path, and the drop-in numerics adapter.
#include <cmath>

#include "common.cuh"
#include "runtime.h"

namespace moe {

__device__ __forceinline__ double dev_round_to(int fmt, double x) {
    if (isnan(x)) return x;
    if (fmt == 0) return (double)(float)x;
    if (x == 0.0 || isinf(x)) return x;
    int mant, emin;
    double maxf;
    bool sat;
    if (fmt == 1) { mant = 7; emin = -126; maxf = ldexp(2.0 - ldexp(1.0, -7), 127); sat = false; }
    else { mant = 3; emin = -6; maxf = 448.0; sat = true; }
    int e = ilogb(fabs(x));
    if (e < emin) e = emin;
    const int q = e - mant;
    const double r = ldexp(rint(ldexp(x, -q)), q);
    if (fabs(r) > maxf) return sat ? copysign(maxf, x) : copysign(__longlong_as_double(0x7ff0000000000000ll), x);
    return r;
}

__device__ __forceinline__ double dev_max_finite(int fmt) {
    if (fmt == 1) return ldexp(2.0 - ldexp(1.0, -7), 127);
    if (fmt == 2) return 448.0;
    return 3.4028234663852886e38;
}

__device__ __forceinline__ int64_t dev_block_of(int gran, int64_t r, int64_t c, int64_t cols, int64_t gs) {
    switch (gran) {
        case 0: return 0;
        case 1: return r;
        case 2: return c;
        default: return r * ((cols + gs - 1) / gs) + c / gs;
    }
}

__global__ void round_kernel(int fmt, const double* __restrict__ x, double* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = dev_round_to(fmt, x[i]);
}

// absmax per block; non-negative doubles order like their bit patterns
__global__ void absmax_kernel(const double* __restrict__ x, int64_t rows, int64_t cols, int gran,
                              int64_t gs, unsigned long long* __restrict__ amax) {
    const int64_t n = rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols, c = i - (i / cols) * cols;
        const double v = fabs(x[i]);
        if (isnan(v)) continue;  // the reference's `v > m` never admits NaN
        atomicMax(&amax[dev_block_of(gran, r, c, cols, gs)], (unsigned long long)__double_as_longlong(v));
    }
}

__global__ void scales_kernel(const unsigned long long* __restrict__ amax, int64_t nb, int fmt,
                              double* __restrict__ scales) {
    const double mf = dev_max_finite(fmt);
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        const double a = __longlong_as_double((long long)amax[b]);
        scales[b] = a > 0.0 ? a / mf : 1.0;
    }
}

__global__ void codes_kernel(const double* __restrict__ x, int64_t rows, int64_t cols, int gran, int64_t gs,
                             int fmt, const double* __restrict__ scales, double* __restrict__ codes) {
    const int64_t n = rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols, c = i - (i / cols) * cols;
        codes[i] = dev_round_to(fmt, x[i] / scales[dev_block_of(gran, r, c, cols, gs)]);
    }
}

__global__ void emulate_reduce_kernel(const double* __restrict__ v, int64_t ranks, int64_t dim, int kind,
                                      double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x) {
        double acc = dev_round_to(1, v[i]);
        for (int64_t r = 1; r < ranks; ++r) {
            acc += dev_round_to(1, v[r * dim + i]);
            if (kind == 0 && r + 1 < ranks) acc = dev_round_to(1, acc);
        }
        out[i] = acc;
    }
}

__global__ void dequantize_kernel(const double* __restrict__ codes, const double* __restrict__ scales,
                                  int64_t rows, int64_t cols, int gran, int64_t gs, double* __restrict__ out) {
    const int64_t n = rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols, c = i - (i / cols) * cols;
        out[i] = codes[i] * scales[dev_block_of(gran, r, c, cols, gs)];
    }
}

// SwiGLU over rows [a | b] in binary64 (numerics.cpp:249-281): out = a * silu(b) (* w[r])
__global__ void swiglu_rows_kernel(const double* __restrict__ x, int64_t rows, int64_t cols,
                                   const double* __restrict__ w, double* __restrict__ out) {
    const int64_t half = cols / 2, n = rows * half;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / half, c = i - r * half;
        const double a = x[r * cols + c], b = x[r * cols + half + c];
        double v = a * (b / (1.0 + exp(-b)));
        if (w) v *= w[r];
        out[i] = v;
    }
}

static int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, kNumSMs * 16)); }

}  // namespace moe

using namespace moe;

extern "C" {

moe_status moe_round_to(int32_t fmt, const double* d_x, int64_t n, double* d_out, moe_stream_t stream) {
    MOE_CHECK_ARG(fmt >= 0 && fmt <= 2, "unknown format");
    MOE_CHECK_ARG(n >= 0, "n must be >= 0");
    if (n == 0) return MOE_OK;
    round_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(fmt, d_x, d_out, n);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

int64_t moe_quantize_num_blocks(int64_t rows, int64_t cols, int32_t gran, int64_t group_size) {
    int64_t nb = 1;
    if (gran == 1) nb = rows;
    else if (gran == 2) nb = cols;
    else if (gran == 3) nb = group_size >= 1 ? rows * ((cols + group_size - 1) / group_size) : 1;
    return nb < 1 ? 1 : nb;
}

size_t moe_quantize_workspace_size(int64_t rows, int64_t cols, int32_t gran, int64_t group_size) {
    const int64_t nb = moe_quantize_num_blocks(rows, cols, gran, group_size);
    return (size_t)std::max<int64_t>(nb, 1) * sizeof(unsigned long long);
}

moe_status moe_quantize(const double* d_x, int64_t rows, int64_t cols, int32_t gran, int64_t group_size,
                        int32_t fmt, double* d_codes, double* d_scales, void* d_workspace,
                        moe_stream_t stream) {
    MOE_CHECK_ARG(rows >= 0 && cols >= 0, "tensor shape does not match data size");
    MOE_CHECK_ARG(!(gran == 3 && group_size < 1), "group_size must be >= 1");
    MOE_CHECK_ARG(gran >= 0 && gran <= 3 && fmt >= 0 && fmt <= 2, "unknown granularity or format");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nb = std::max<int64_t>(moe_quantize_num_blocks(rows, cols, gran, group_size), 1);
    auto* amax = static_cast<unsigned long long*>(d_workspace);
    MOE_CUDA_TRY(cudaMemsetAsync(amax, 0, nb * sizeof(unsigned long long), s));
    const int64_t n = rows * cols;
    if (n > 0) {
        absmax_kernel<<<grid_for(n), 256, 0, s>>>(d_x, rows, cols, gran, group_size, amax);
        count_launch();
    }
    scales_kernel<<<grid_for(nb), 256, 0, s>>>(amax, nb, fmt, d_scales);
    count_launch();
    if (n > 0) {
        codes_kernel<<<grid_for(n), 256, 0, s>>>(d_x, rows, cols, gran, group_size, fmt, d_scales, d_codes);
        count_launch();
    }
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

moe_status moe_dequantize(const double* d_codes, const double* d_scales, int64_t rows, int64_t cols,
                          int32_t gran, int64_t group_size, double* d_out, moe_stream_t stream) {
    MOE_CHECK_ARG(rows >= 0 && cols >= 0 && gran >= 0 && gran <= 3, "bad shape or granularity");
    if (rows * cols == 0) return MOE_OK;
    dequantize_kernel<<<grid_for(rows * cols), 256, 0, (cudaStream_t)stream>>>(d_codes, d_scales, rows, cols,
                                                                               gran, group_size, d_out);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

moe_status moe_swiglu_rows_f64(const double* d_x, int64_t rows, int64_t cols, const double* d_row_weight,
                               double* d_out, moe_stream_t stream) {
    MOE_CHECK_ARG(cols % 2 == 0, "cols must be even: rows are [a | b] pairs");
    if (rows * cols == 0) return MOE_OK;
    swiglu_rows_kernel<<<grid_for(rows * cols / 2), 256, 0, (cudaStream_t)stream>>>(d_x, rows, cols,
                                                                                    d_row_weight, d_out);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

moe_status moe_emulate_reduce(const double* d_vectors, int64_t ranks, int64_t dim, int32_t kind,
                              double* d_out, moe_stream_t stream) {
    MOE_CHECK_ARG(ranks >= 2, "reduction needs at least 2 ranks");
    MOE_CHECK_ARG(kind == 0 || kind == 1, "unknown reduce scheme");
    if (dim == 0) return MOE_OK;
    emulate_reduce_kernel<<<grid_for(dim), 256, 0, (cudaStream_t)stream>>>(d_vectors, ranks, dim, kind, d_out);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

}  // extern "C"
