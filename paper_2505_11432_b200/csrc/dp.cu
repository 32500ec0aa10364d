// dp.cu — data-parallel gradient synchronisation with BF16 communication
// compression (the paper's DP compression; cost model
// commcost.cpp:182-201, memory model memmodel.cpp:112-114):
//
//   reduce-scatter:  the fp32 main gradient [count] is cast to BF16 IN PLACE
//                    into the low half of its own buffer; every rank then pulls
//                    its shard's BF16 pieces from all peers over NVLink
//                    (all-to-all) and sums them in rank order with a wide
//                    accumulator (a2a_fp32 semantics, numerics.cpp:172-192:
//                    inputs rounded to bf16 once, no bf16 re-rounding between
//                    ranks). The fp32 shard lands in the high half of the same
//                    buffer, so the operator needs no memory beyond the fp32
//                    gradient itself (the reference's transient_peak is 0 for
//                    the in-place operator, grads/2 for the naive one).
//   all-gather:      the updated fp32 shard is cast to BF16 and every rank
//                    pulls all shards.
// Bytes on the wire per rank: (n-1)/n * count * 2 per collective, half of an
// fp32 reduce-scatter.
#include <cstring>
#include <vector>

#include "common.cuh"
#include "layer_kernels.cuh"
#include "runtime.h"

using namespace moe;

struct moe_dp {
    int64_t count = 0, n = 1, rank = 0, shard = 0, nchunks = 0;
    uint8_t* arena = nullptr;
    size_t off_flags = 0, arena_bytes = 0;
    std::vector<uint8_t*> peer;
    void** tab = nullptr;          // [2][n]: buffers, flags
    uint32_t* chunk_flag = nullptr;  // in-place cast progress [nchunks]
    uint32_t* epoch_dev = nullptr;
    int* err = nullptr;
    bool ipc_ready = false;
};

namespace {

constexpr int kCastThreads = 256;
constexpr int kCastVec = 4;                                   // float4 per thread per chunk
constexpr int64_t kChunk = kCastThreads * kCastVec * 4;       // 4096 floats per chunk

template <class T>
moe_status dalloc(T** p, size_t count) {
    MOE_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T)));
    return MOE_OK;
}

// In-place fp32 -> bf16 cast into the low half of the same buffer. Chunk c
// (fp32 elements [c*CH, (c+1)*CH)) writes bf16 bytes [2c*CH, 2(c+1)*CH), which
// overlap exactly the fp32 input of chunk c/2; so chunk c publishes "read" once
// its input is in registers and writes only after chunk c/2 has published.
// Dependencies point to strictly lower chunks and chunks are claimed in
// increasing order from a counter (chunk_flag[nchunks]) by whichever CTA asks
// next, so the chunk a CTA waits for is held by a CTA that is already running:
// no deadlock whatever part of the grid is resident.
__global__ void __launch_bounds__(kCastThreads) dp_cast_inplace_kernel(float* buf, int64_t nchunks,
                                                                        uint32_t* chunk_flag, int* err) {
    __shared__ int64_t s_c;
    for (;;) {
        if (threadIdx.x == 0) s_c = (int64_t)atomicAdd(&chunk_flag[nchunks], 1u);
        __syncthreads();
        const int64_t c = s_c;
        if (c >= nchunks) break;
        const float4* src = reinterpret_cast<const float4*>(buf + c * kChunk);
        uint32_t pk[kCastVec][2];
#pragma unroll
        for (int v = 0; v < kCastVec; ++v) {
            const float4 f = src[v * kCastThreads + threadIdx.x];
            pk[v][0] = pack_bf16x2(f.x, f.y);
            pk[v][1] = pack_bf16x2(f.z, f.w);
        }
        __syncthreads();   // every thread of this CTA has its chunk in registers
        if (threadIdx.x == 0) {
            __threadfence();
            red_release_gpu_add(&chunk_flag[c], 1u);
            if (c > 0) {
                const uint64_t t0 = globaltimer();
                while (ld_acquire_gpu(&chunk_flag[c / 2]) == 0u) {
                    if (globaltimer() - t0 > 4000000000ull) { atomicExch(err, 3); break; }
                }
            }
        }
        __syncthreads();
        uint2* dst = reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(buf) + c * kChunk);
#pragma unroll
        for (int v = 0; v < kCastVec; ++v) dst[v * kCastThreads + threadIdx.x] = make_uint2(pk[v][0], pk[v][1]);
        __syncthreads();  // s_c is reused by the next claim
    }
}

// Shard reduction: out[i] = (float) sum_p bf16(peer_p[r*S + i]) in rank order,
// accumulated in binary64 (exactly the reference's emulate_reduce(a2a_fp32)
// followed by one cast to fp32). 8 elements (16 B per peer) per thread-step.
__global__ void dp_a2a_reduce_kernel(const uint16_t* const* bufs, int n, int64_t base, int64_t S,
                                     float* __restrict__ out) {
    const int64_t nv = S / 8;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        double acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = -0.0;   // -0 + v == v exactly (keeps -0 sums)
        uint4 q[8];
        for (int p0 = 0; p0 < n; p0 += 8) {
            const int np = n - p0 < 8 ? n - p0 : 8;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < np) q[j] = reinterpret_cast<const uint4*>(bufs[p0 + j] + base)[v];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j < np) {
                    const uint32_t w[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f = unpack_bf16x2(w[e]);
                        acc[2 * e] += (double)f.x;
                        acc[2 * e + 1] += (double)f.y;
                    }
                }
            }
        }
        float4* o = reinterpret_cast<float4*>(out + v * 8);
        o[0] = make_float4((float)acc[0], (float)acc[1], (float)acc[2], (float)acc[3]);
        o[1] = make_float4((float)acc[4], (float)acc[5], (float)acc[6], (float)acc[7]);
    }
}

// n = 1: the "reduction" is the bf16 round trip of every element, in place.
__global__ void dp_round_bf16_kernel(float* buf, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count / 4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 f = reinterpret_cast<float4*>(buf)[i];
        const float2 a = unpack_bf16x2(pack_bf16x2(f.x, f.y)), b = unpack_bf16x2(pack_bf16x2(f.z, f.w));
        reinterpret_cast<float4*>(buf)[i] = make_float4(a.x, a.y, b.x, b.y);
    }
}

__global__ void dp_cast_shard_kernel(const float* __restrict__ src, uint16_t* __restrict__ dst, int64_t S) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S / 4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 f = reinterpret_cast<const float4*>(src)[i];
        reinterpret_cast<uint2*>(dst)[i] = make_uint2(pack_bf16x2(f.x, f.y), pack_bf16x2(f.z, f.w));
    }
}

// out[p*S + i] = peer_p[p*S + i] (bf16), all peers; 8 independent 16 B loads
// in flight per thread (peer reads over NVLink are latency-bound otherwise),
// peers visited starting from this rank so the links are loaded evenly
__global__ void dp_gather_kernel(const uint16_t* const* bufs, int n, int rank, int64_t S, uint16_t* __restrict__ out) {
    constexpr int U = 8;
    const int64_t nv = S / 8;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int j = 0; j < n; ++j) {
        const int p = (rank + j) % n;
        const uint4* src = reinterpret_cast<const uint4*>(bufs[p]) + p * nv;
        uint4* dst = reinterpret_cast<uint4*>(out) + p * nv;
        for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < nv; v0 += stride * U) {
            uint4 r[U];
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (v0 + q * stride < nv) r[q] = src[v0 + q * stride];
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (v0 + q * stride < nv) dst[v0 + q * stride] = r[q];
        }
    }
}

moe_status fill(moe_dp* D) {
    const int n = (int)D->n;
    std::vector<void*> t(2 * n);
    for (int p = 0; p < n; ++p) {
        t[p] = D->peer[p];
        t[n + p] = D->peer[p] + D->off_flags;
    }
    MOE_CUDA_TRY(cudaMemcpy(D->tab, t.data(), sizeof(void*) * t.size(), cudaMemcpyHostToDevice));
    return MOE_OK;
}

moe_status dp_barrier(moe_dp* D, int slot, cudaStream_t s) {
    if (D->n == 1) return MOE_OK;
    flag_barrier_kernel<<<1, 64, 0, s>>>(reinterpret_cast<uint32_t* const*>(D->tab + D->n), slot, (int)D->n,
                                        (int)D->rank, D->epoch_dev, 1, flag_timeout_ns(), D->err);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

int grid_for(int64_t work) { return (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, kNumSMs * 8)); }

}  // namespace

extern "C" {

moe_status moe_dp_create(int64_t count, int64_t dp_size, int64_t rank, moe_dp** out) {
    MOE_CHECK_ARG(out, "null argument");
    MOE_CHECK_ARG(dp_size >= 1 && dp_size <= 64 && rank >= 0 && rank < dp_size, "bad dp_size/rank");
    MOE_CHECK_ARG(count > 0 && count % (kChunk * dp_size) == 0,
                  "count must be a positive multiple of 4096 * dp_size");
    auto* D = new moe_dp();
    D->count = count;
    D->n = dp_size;
    D->rank = rank;
    D->shard = count / dp_size;
    D->nchunks = count / kChunk;
    D->off_flags = (size_t)count * 4;
    D->arena_bytes = D->off_flags + 16 * 64 * 4;
    moe_status st;
#define TRY(expr) do { st = (expr); if (st != MOE_OK) { moe_dp_destroy(D); return st; } } while (0)
    TRY(dalloc(&D->arena, D->arena_bytes));
    cudaMemset(D->arena, 0, D->arena_bytes);
    D->peer.assign(D->n, nullptr);
    D->peer[D->rank] = D->arena;
    TRY(dalloc(&D->tab, 2 * D->n));
    TRY(dalloc(&D->chunk_flag, D->nchunks + 1));  // + the chunk-claim counter
    TRY(dalloc(&D->epoch_dev, 1));
    TRY(dalloc(&D->err, 1));
    cudaMemset(D->epoch_dev, 0, 4);
    cudaMemset(D->err, 0, 4);
    if (D->n == 1) {
        TRY(fill(D));
        D->ipc_ready = true;
    }
#undef TRY
    if (cudaDeviceSynchronize() != cudaSuccess) {
        moe_dp_destroy(D);
        return set_error(MOE_ERR_CUDA, "dp init failed");
    }
    *out = D;
    return MOE_OK;
}

void moe_dp_destroy(moe_dp* D) {
    if (!D) return;
    cudaDeviceSynchronize();
    for (int p = 0; p < (int)D->peer.size(); ++p)
        if (p != D->rank && D->peer[p]) cudaIpcCloseMemHandle(D->peer[p]);
    void* bufs[] = {D->arena, D->tab, D->chunk_flag, D->epoch_dev, D->err};
    for (void* b : bufs)
        if (b) cudaFree(b);
    delete D;
}

float* moe_dp_grad_buffer(moe_dp* D) { return D ? reinterpret_cast<float*>(D->arena) : nullptr; }

float* moe_dp_shard(moe_dp* D) {
    if (!D) return nullptr;
    return reinterpret_cast<float*>(D->arena) + (D->n == 1 ? 0 : D->count / 2);
}

moe_status moe_dp_reduce_scatter(moe_dp* D, moe_stream_t stream) {
    MOE_CHECK_ARG(D, "null argument");
    MOE_CHECK_ARG(D->ipc_ready, "dp_size > 1 requires moe_dp_ipc_import");
    cudaStream_t s = (cudaStream_t)stream;
    float* buf = reinterpret_cast<float*>(D->arena);
    if (D->n == 1) {
        dp_round_bf16_kernel<<<grid_for(D->count / 4), 256, 0, s>>>(buf, D->count);
        count_launch();
        MOE_CUDA_TRY(cudaGetLastError());
        return MOE_OK;
    }
    MOE_CUDA_TRY(cudaMemsetAsync(D->chunk_flag, 0, (D->nchunks + 1) * 4, s));
    dp_cast_inplace_kernel<<<(unsigned)std::min<int64_t>(D->nchunks, kNumSMs * 4), kCastThreads, 0, s>>>(
        buf, D->nchunks, D->chunk_flag, D->err);
    count_launch();
    MOE_TRY(dp_barrier(D, 0, s));   // every rank's bf16 copy is in place
    dp_a2a_reduce_kernel<<<grid_for(D->shard / 8), 256, 0, s>>>(
        reinterpret_cast<const uint16_t* const*>(D->tab), (int)D->n, D->rank * D->shard, D->shard,
        buf + D->count / 2);
    count_launch();
    MOE_TRY(dp_barrier(D, 1, s));   // peers are done reading this rank's bf16 half
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

moe_status moe_dp_all_gather_bf16(moe_dp* D, const float* d_shard, uint16_t* d_full, moe_stream_t stream) {
    MOE_CHECK_ARG(D && d_shard && d_full, "null argument");
    MOE_CHECK_ARG(D->ipc_ready, "dp_size > 1 requires moe_dp_ipc_import");
    cudaStream_t s = (cudaStream_t)stream;
    uint16_t* lo = reinterpret_cast<uint16_t*>(D->arena);
    dp_cast_shard_kernel<<<grid_for(D->shard / 4), 256, 0, s>>>(d_shard, lo + D->rank * D->shard, D->shard);
    count_launch();
    MOE_TRY(dp_barrier(D, 2, s));
    dp_gather_kernel<<<kNumSMs * 4, 256, 0, s>>>(reinterpret_cast<const uint16_t* const*>(D->tab), (int)D->n,
                                                (int)D->rank, D->shard, d_full);
    count_launch();
    MOE_TRY(dp_barrier(D, 3, s));
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

size_t moe_dp_ipc_handle_size(void) { return sizeof(cudaIpcMemHandle_t); }

moe_status moe_dp_ipc_export(moe_dp* D, void* h_blob) {
    MOE_CHECK_ARG(D && h_blob, "null argument");
    cudaIpcMemHandle_t hd;
    MOE_CUDA_TRY(cudaIpcGetMemHandle(&hd, D->arena));
    std::memcpy(h_blob, &hd, sizeof(hd));
    return MOE_OK;
}

moe_status moe_dp_ipc_import(moe_dp* D, const void* h_blobs) {
    MOE_CHECK_ARG(D && h_blobs, "null argument");
    const auto* hs = static_cast<const cudaIpcMemHandle_t*>(h_blobs);
    for (int p = 0; p < (int)D->n; ++p) {
        if (p == D->rank) continue;
        void* ptr = nullptr;
        MOE_CUDA_TRY(cudaIpcOpenMemHandle(&ptr, hs[p], cudaIpcMemLazyEnablePeerAccess));
        D->peer[p] = static_cast<uint8_t*>(ptr);
    }
    MOE_TRY(fill(D));
    D->ipc_ready = true;
    return MOE_OK;
}

moe_status moe_dp_status(moe_dp* D, moe_stream_t stream) {
    MOE_CHECK_ARG(D, "null argument");
    return flag_status(D->err, (cudaStream_t)stream, "moe_dp");
}

int moe_dp_error_flag(moe_dp* D) {
    int v = 0;
    if (D && D->err) cudaMemcpy(&v, D->err, sizeof(int), cudaMemcpyDeviceToHost);
    return v;
}

}  // extern "C"
