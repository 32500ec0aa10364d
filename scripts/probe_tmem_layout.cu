// probe_tmem_layout.cu — measures where a cta_group::2 UMMA puts the
// accumulator rows / columns in each CTA's TMEM for M = 256 and M = 128
// (development probe; the grouped GEMM's tail tiles rely on the M = 128 map).
//   A[r][0] = r + 1 (global row), A[r][1] = 1024;  B[n][0] = 1, B[n][1] = n + 1
//   => D[r][n] = (r + 1) + 1024 (n + 1), decodable from every TMEM word.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I. scripts/probe_tmem_layout.cu -o /tmp/probe
#include <cstdio>
#include <vector>

#include "paper_2505_11432_b200/csrc/gemm_sm100.cuh"

using namespace moe;

constexpr int N = 128;
constexpr int COLS = 256;

__device__ void put(uint8_t* tile, int r, int kk, float v) {
    const int off = (r / 8) * 1024 + (r % 8) * 128 + (((kk / 8) ^ (r % 8)) * 16) + (kk % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(tile + off) = __float2bfloat16(v);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(int M, uint32_t* out) {
    __shared__ __align__(1024) uint8_t sA[16384];
    __shared__ __align__(1024) uint8_t sB[16384];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t cta = cluster_ctarank();
    const int tid = threadIdx.x, warp = tid / 32;
    for (int i = tid; i < 16384 / 4; i += 128) {
        reinterpret_cast<uint32_t*>(sA)[i] = 0;
        reinterpret_cast<uint32_t*>(sB)[i] = 0;
    }
    __syncthreads();
    const int rows_per_cta = M / 2;
    for (int r = tid; r < 128; r += 128) {
        if (r < rows_per_cta) {
            put(sA, r, 0, (float)(cta * rows_per_cta + r + 1));
            put(sA, r, 1, 1024.0f);
        }
        if (r < N / 2) {
            put(sB, r, 0, 1.0f);
            put(sB, r, 1, (float)(cta * (N / 2) + r + 1));
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc_2sm<COLS>(&tslot);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tbase = tslot;
    if (cta == 0 && tid == 0) {
        const uint64_t ad = make_sdesc(smem_u32(sA), 16, 1024);
        const uint64_t bd = make_sdesc(smem_u32(sB), 16, 1024);
        const uint32_t idesc = make_idesc(M, N, 1, false, false);
        umma_bf16_2sm(tbase, ad, bd, idesc, 0u);
        umma_commit_2sm_mc(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    for (int c0 = 0; c0 < COLS; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + c0, r);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) out[((size_t)cta * 128 + tid) * COLS + c0 + j] = r[j];
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 0) tmem_dealloc_2sm<COLS>(tbase);
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 2 * 128 * COLS * 4);
    std::vector<uint32_t> h(2 * 128 * COLS);
    for (int M : {256, 128}) {
        cudaMemset(d, 0, h.size() * 4);
        probe<<<2, 128>>>(M, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("M=%d error %s\n", M, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
        char fn[64];
        snprintf(fn, sizeof fn, "gpurun_out/tmem_M%d.bin", M);
        FILE* fp = fopen(fn, "wb");
        fwrite(h.data(), 4, h.size(), fp);
        fclose(fp);
    }
    return 0;
}
