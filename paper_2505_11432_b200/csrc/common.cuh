// common.cuh — sm_100a device helpers shared by every kernel of the MoE hot
// path: mbarrier / TMA / tcgen05 (UMMA, TMEM) inline PTX, bf16 and e4m3
// conversions, and the status plumbing behind the C ABI.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/moe_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "this library targets sm_100a only"
#endif

namespace moe {

// ---------------------------------------------------------------------------
// host-side status
// ---------------------------------------------------------------------------
moe_status set_error(moe_status st, const char* fmt, ...);

#define MOE_CUDA_TRY(expr)                                                          \
    do {                                                                            \
        cudaError_t _e = (expr);                                                    \
        if (_e != cudaSuccess)                                                      \
            return ::moe::set_error(MOE_ERR_CUDA, "%s failed: %s (%s:%d)", #expr,   \
                                    cudaGetErrorString(_e), __FILE__, __LINE__);    \
    } while (0)

#define MOE_CHECK_ARG(cond, msg)                                                    \
    do {                                                                            \
        if (!(cond)) return ::moe::set_error(MOE_ERR_INVALID, "%s", msg);           \
    } while (0)

#define MOE_TRY(expr)                                                               \
    do {                                                                            \
        moe_status _s = (expr);                                                     \
        if (_s != MOE_OK) return _s;                                                \
    } while (0)

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

// --- mbarrier --------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// --- TMA -------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map,
                                            uint64_t* bar, int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// generic-proxy writes (ld/st from other SMs or peers) -> async proxy (TMA)
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// --- tcgen05 / TMEM ----------------------------------------------------------
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate.
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// tf32 inputs (fp32 storage), fp32 accumulate.
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05.mma of this
// thread have completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns; thread i gets lane (base+i).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory matrix descriptor (Blackwell "version 1"), 128B swizzle.
//   K-major operand: rows of 128 B (64 bf16 of K), 8-row groups 1024 B apart
//                    (SBO); LBO unused (1).
//   MN-major operand: 128 B of MN (64 bf16) per K row, 8 K rows per 1024 B
//                    atom (SBO = 1024 B between 8-row K groups), LBO = byte
//                    distance between 64-element MN chunks.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t smem_addr, uint32_t lbo_bytes,
                                               uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // descriptor version (sm_100)
    d |= 2ull << 61;  // SWIZZLE_128B
    return d;
}

// Instruction descriptor for kind::f16 / kind::tf32 with fp32 accumulate.
//   fmt: 0 f16, 1 bf16, 2 tf32.
__host__ __device__ constexpr uint32_t make_idesc(uint32_t M, uint32_t N, uint32_t fmt,
                                                  bool a_mn_major, bool b_mn_major) {
    return (1u << 4)                                  // D = f32
           | (fmt << 7) | (fmt << 10)                 // A, B format
           | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
           ((N >> 3) << 17) | ((M >> 4) << 24);
}

// ---------------------------------------------------------------------------
// numeric helpers
// ---------------------------------------------------------------------------
// sigmoid via ex2.approx + rcp.approx (rcp of +inf is 0, so large negative
// inputs give 0); the SwiGLU epilogues (fwd and bwd) share it, so the bwd
// remat of fc2_in reproduces the forward values bit for bit
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sigmoid_f(float v) { return rcp_approx(1.0f + __expf(-v)); }
__device__ __forceinline__ float silu_f(float v) { return v * sigmoid_f(v); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float2 unpack_bf16x2(uint32_t v) {
    __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&v);
    return __bfloat1622float2(b);
}

// E4M3 pack/unpack (RNE, saturating to +-448; the FP8 communication format,
// PAPER.md:359-360). lo goes to the low byte.
__device__ __forceinline__ uint16_t f32x2_to_e4m3x2(float lo, float hi) {
    uint16_t r;
    asm("{cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;}" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ float2 e4m3x2_to_f32x2(uint16_t v) {
    uint32_t h2;
    asm("{cvt.rn.f16x2.e4m3x2 %0, %1;}" : "=r"(h2) : "h"(v));
    __half2 hh = *reinterpret_cast<__half2*>(&h2);
    return __half22float2(hh);
}

// E4M3 code of a binary64 value with RNE + saturation at 448 and the 2^-9
// subnormal quantum (numerics.cpp:50-68), computed in binary64 so no
// intermediate rounding can move a value across a rounding midpoint.
__device__ __forceinline__ uint8_t e4m3_rne_code(double q) {
    if (q != q) return 0x7f;  // NaN
    if (q == 0.0) return signbit(q) ? 0x80 : 0x00;
    const double aq = fabs(q);
    int e = ilogb(aq);
    if (e < -6) e = -6;  // subnormal range: quantum 2^-9
    const double quantum = ldexp(1.0, e - 3);
    double r = rint(aq / quantum) * quantum;  // exact: division by a power of two
    if (r > 448.0) r = 448.0;                 // saturate (numerics.cpp:63-65)
    uint8_t code;
    if (r < ldexp(1.0, -6)) {
        code = (uint8_t)(int)(r / ldexp(1.0, -9));  // subnormal mantissa 0..7
    } else {
        const int ee = ilogb(r);
        const int mant = (int)(r / ldexp(1.0, ee - 3)) - 8;
        code = (uint8_t)(((ee + 7) << 3) | mant);
    }
    return (uint8_t)(code | (q < 0 ? 0x80 : 0));
}

// Block quantiser with the reference's arithmetic (numerics.cpp:149-156):
// scale = absmax / 448 and code = E4M3(x / scale), both in binary64. The
// hot kernels take a fast path — x * (1/scale rounded to fp32), two fp32
// roundings, relative error < 2^-23 — and fall back to the binary64 division
// when that quotient lies within 2^-16 quanta of an E4M3 rounding midpoint,
// the only place the two can round differently (a quantum is >= 2^-20 of the
// quotient's magnitude, so 2^-16 quanta is >= 8 fp32 ulps of margin). Codes
// are therefore bit-identical to the reference for every fp32 / bf16 input.
// The stored scale is the binary64 scale rounded once to fp32.
struct E4m3Block {
    double scale;  // binary64 scale (absmax / 448, or 1 for an all-zero block)
    float inv;     // 1 / scale rounded to fp32
    bool exact;    // 1 / scale overflows fp32 (absmax < ~1.3e-36): always divide
};
__device__ __forceinline__ E4m3Block e4m3_block(float amax) {
    E4m3Block b;
    b.scale = amax > 0.0f ? (double)amax / 448.0 : 1.0;
    const double inv = 1.0 / b.scale;
    b.exact = inv > 3.0e38;
    b.inv = b.exact ? 0.0f : (float)inv;
    return b;
}
// true when |q| (fp32) is within 2^-16 quanta of an E4M3 rounding midpoint
__device__ __forceinline__ bool e4m3_near_midpoint(float q) {
    const uint32_t bits = __float_as_uint(q) & 0x7fffffffu;
    int e = (int)(bits >> 23) - 127;
    if (e < -6) e = -6;
    // t = |q| / quantum, quantum = 2^(e-3): exact power-of-two scaling
    const float t = __uint_as_float(bits) * __uint_as_float((uint32_t)(127 - (e - 3)) << 23);
    return fabsf(t - floorf(t) - 0.5f) < 1.52587890625e-5f;  // 2^-16
}
__device__ __forceinline__ uint8_t e4m3_code(float x, const E4m3Block& b) {
    if (b.exact) return e4m3_rne_code((double)x / b.scale);
    const float q = x * b.inv;
    if (e4m3_near_midpoint(q) && fabsf(q) < 464.0f) return e4m3_rne_code((double)x / b.scale);
    return (uint8_t)(f32x2_to_e4m3x2(q, 0.0f) & 0xff);
}
// two codes packed (lo = first), fast path through one cvt
__device__ __forceinline__ uint16_t e4m3x2_code(float x0, float x1, const E4m3Block& b) {
    if (!b.exact) {
        const float q0 = x0 * b.inv, q1 = x1 * b.inv;
        const bool n0 = e4m3_near_midpoint(q0) && fabsf(q0) < 464.0f;
        const bool n1 = e4m3_near_midpoint(q1) && fabsf(q1) < 464.0f;
        if (!(n0 | n1)) return f32x2_to_e4m3x2(q0, q1);
    }
    return (uint16_t)e4m3_code(x0, b) | ((uint16_t)e4m3_code(x1, b) << 8);
}

// --- system-scope flags for cross-GPU signalling ----------------------------
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_sys_add(uint32_t* p, uint32_t v) {
    asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

}  // namespace moe
