// quant.cu — per-token (1 x h) E4M3 quantisation for FP8 dispatch/combine
// communication (reference numerics.cpp:113-160 with
// Granularity::per_token, Format::fp8_e4m3).
//
// Bit-exactness: the reference computes scale = absmax / 448 and
// x / scale in binary64 and rounds to E4M3 with RNE + saturation
// (numerics.cpp:50-68). This kernel does the same arithmetic in fp64 on the
// device, so codes match the reference bit for bit on fp32/bf16 inputs; the
// scale is stored as fp32 (its binary64 value rounded once).
#include "common.cuh"
#include "runtime.h"

namespace moe {

// e4m3_rne_code (binary64 RNE + saturation) lives in common.cuh: the
// layer's hot quantisers fall back to it near rounding midpoints.

template <bool F32>
__global__ void quantize_rows_kernel(const void* __restrict__ xv, int cols,
                                     uint8_t* __restrict__ codes, float* __restrict__ scales) {
    const int64_t row = blockIdx.x;
    __shared__ float s_red[32];
    float m = 0.0f;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
        float v;
        if (F32) v = static_cast<const float*>(xv)[row * cols + c];
        else v = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(xv)[row * cols + c]);
        m = fmaxf(m, fabsf(v));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? s_red[threadIdx.x] : 0.0f;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
        if (threadIdx.x == 0) s_red[0] = v;
    }
    __syncthreads();
    const double absmax = (double)s_red[0];
    const double scale = absmax > 0.0 ? absmax / 448.0 : 1.0;
    if (threadIdx.x == 0) scales[row] = (float)scale;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
        double v;
        if (F32) v = (double)static_cast<const float*>(xv)[row * cols + c];
        else v = (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(xv)[row * cols + c]);
        codes[row * cols + c] = e4m3_rne_code(v / scale);
    }
}

moe_status launch_quantize_e4m3_rows(const void* x, bool x_is_f32, int64_t rows, int64_t cols,
                                     uint8_t* codes, float* scales, cudaStream_t s) {
    MOE_CHECK_ARG(rows >= 0 && cols >= 0, "tensor shape does not match data size");
    if (rows == 0 || cols == 0) return MOE_OK;
    MOE_CHECK_ARG(rows < (1ll << 31), "too many rows");
    if (x_is_f32)
        quantize_rows_kernel<true><<<(unsigned)rows, 256, 0, s>>>(x, (int)cols, codes, scales);
    else
        quantize_rows_kernel<false><<<(unsigned)rows, 256, 0, s>>>(x, (int)cols, codes, scales);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

}  // namespace moe
