// gemm.cu — host launchers for the tcgen05 grouped GEMM (gemm_sm100.cuh)
// and the C-ABI `moe_grouped_gemm` operator (reference OpKind::grouped_gemm,
// simsched.hpp:32-44).
#include <atomic>
#include <cstdlib>
#include <mutex>

#include "gemm.h"

namespace moe {

// Dynamic tile schedule counters of the stateless operators (moe_grouped_gemm):
// one int per launch from a per-device ring, zeroed on the launch's stream
// just before it. A slot is reused only after kCounters later launches, so do
// not keep a graph that captured moe_grouped_gemm while issuing thousands of
// eager ones concurrently. Layer / attention / Ulysses plans own their
// counters (GemmPlan::counter).
static int* tile_counter_slot(int dev) {
    constexpr int kDevices = 64, kCounters = 4096;
    static int* base[kDevices] = {};
    static std::atomic<unsigned> next[kDevices];
    static std::mutex mu;
    if (dev < 0 || dev >= kDevices) return nullptr;
    if (!base[dev]) {
        std::lock_guard<std::mutex> lock(mu);
        if (!base[dev] && cudaMalloc(&base[dev], kCounters * sizeof(int)) != cudaSuccess) return nullptr;
    }
    return base[dev] + (next[dev].fetch_add(1) % kCounters);
}

template <int BN, int CG, bool A_MN, bool B_MN, bool KG, int EPI, bool DISP = false>
static moe_status launch_impl(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a,
                              int grid, cudaStream_t s) {
    using Cfg = GemmCfg<BN, CG>;
    auto kern = grouped_gemm_kernel<BN, CG, A_MN, B_MN, KG, EPI, DISP>;
    constexpr int kThreads = Cfg::THREADS + (DISP ? 32 * Cfg::COMM_WARPS : 0) + (EPI == EPI_SCATTER_RS ? 32 : 0);
    static uint64_t attr_set = 0;  // per instantiation, one bit per device
    int dev = 0;
    MOE_CUDA_TRY(cudaGetDevice(&dev));
    if (!(attr_set >> (dev & 63) & 1)) {
        MOE_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          Cfg::SMEM_BYTES));
        attr_set |= 1ull << (dev & 63);
    }
    if (CG == 1) {
        kern<<<grid, kThreads, Cfg::SMEM_BYTES, s>>>(ta, tb, a);
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(grid & ~1));
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        MOE_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, a));
    }
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

moe_status gemm_launch(const GemmPlan& p, const GemmArgs& args, cudaStream_t s) {
    MOE_CHECK_ARG(args.G >= 1 && args.G <= 256, "grouped GEMM: 1 <= groups <= 256");
    const int grid = p.grid > 0 ? p.grid : kNumSMs;
    GemmArgs a = args;
    static const bool static_tiles = getenv("MOE_STATIC_TILES") != nullptr;
    // (the kernel keeps the static stride for K-grouped and multi-group K >= 8192 GEMMs)
    if (!a.tile_counter && !static_tiles && !p.k_grouped && (a.K < 8192 || a.G == 1)) {
        if (p.counter) {
            a.tile_counter = p.counter;
        } else {
            int dev = 0;
            MOE_CUDA_TRY(cudaGetDevice(&dev));
            a.tile_counter = tile_counter_slot(dev);
        }
        if (a.tile_counter) MOE_CUDA_TRY(cudaMemsetAsync(a.tile_counter, 0, sizeof(int), s));
    }
#define MOE_GEMM_CASE(BN, CG, AMN, BMN, KG, EPI)                                              \
    if (p.bn == BN && p.cg == CG && p.a_mn == AMN && p.b_mn == BMN && p.k_grouped == KG &&   \
        p.epi == EPI && !p.dispatch)                                                          \
        return launch_impl<BN, CG, AMN, BMN, KG, EPI>(p.ta, p.tb, a, grid, s);
#define MOE_GEMM_CASE_DISP(BN, CG, AMN, BMN, KG, EPI)                                         \
    if (p.bn == BN && p.cg == CG && p.a_mn == AMN && p.b_mn == BMN && p.k_grouped == KG &&   \
        p.epi == EPI && p.dispatch)                                                           \
        return launch_impl<BN, CG, AMN, BMN, KG, EPI, true>(p.ta, p.tb, a, grid, s);
    // fused AG + scatter + GroupedGEMM (fc1 forward, fc2 dgrad)
    MOE_GEMM_CASE_DISP(256, 2, false, false, false, EPI_SWIGLU)
    MOE_GEMM_CASE_DISP(256, 2, false, true, false, EPI_SWIGLU_BWD)
    MOE_GEMM_CASE_DISP(256, 1, false, false, false, EPI_SWIGLU)
    MOE_GEMM_CASE_DISP(256, 1, false, true, false, EPI_SWIGLU_BWD)
    MOE_GEMM_CASE_DISP(256, 2, false, false, false, EPI_STORE_BF16)  // attention AG-GEMM
    MOE_GEMM_CASE_DISP(256, 1, false, false, false, EPI_STORE_BF16)
    MOE_GEMM_CASE_DISP(128, 2, false, false, false, EPI_STORE_BF16)  // AG-GEMM, 256 x 128 pair tiles
    // layer GEMMs, CTA-pair (cta_group::2) versions
    MOE_GEMM_CASE(256, 2, false, false, false, EPI_SWIGLU)       // fc1 + SwiGLU
    MOE_GEMM_CASE(256, 2, false, false, false, EPI_SCATTER)      // fc2 + gather
    MOE_GEMM_CASE(256, 2, false, true, false, EPI_SWIGLU_BWD)    // fc2 dgrad
    MOE_GEMM_CASE(256, 2, false, true, false, EPI_SCATTER)       // fc1 dgrad
    MOE_GEMM_CASE(256, 2, false, false, false, EPI_SCATTER_FP8)  // fc2 + FP8 combine payload
    MOE_GEMM_CASE(256, 2, false, false, false, EPI_SCATTER_RS)   // TP GEMM-RS, fused reduce
    MOE_GEMM_CASE(256, 2, false, true, false, EPI_SCATTER_FP8)   // fc1 dgrad + FP8 payload
    MOE_GEMM_CASE(256, 2, true, true, true, EPI_STORE_BF16)      // wgrads
    MOE_GEMM_CASE(256, 2, true, true, true, EPI_STORE_F32)
    MOE_GEMM_CASE(256, 2, false, false, false, EPI_STORE_BF16)   // generic
    MOE_GEMM_CASE(256, 2, false, false, false, EPI_STORE_F32)
    MOE_GEMM_CASE(256, 2, false, true, false, EPI_STORE_F32)
    MOE_GEMM_CASE(256, 2, false, true, false, EPI_STORE_BF16)
    // single-CTA versions
    MOE_GEMM_CASE(256, 1, false, false, false, EPI_SWIGLU)
    MOE_GEMM_CASE(256, 1, false, false, false, EPI_SCATTER)
    MOE_GEMM_CASE(256, 1, false, false, false, EPI_SCATTER_FP8)
    MOE_GEMM_CASE(256, 1, false, false, false, EPI_SCATTER_RS)
    MOE_GEMM_CASE(256, 1, false, true, false, EPI_SCATTER_FP8)
    MOE_GEMM_CASE(256, 1, false, true, false, EPI_SWIGLU_BWD)
    MOE_GEMM_CASE(256, 1, false, true, false, EPI_SCATTER)
    MOE_GEMM_CASE(256, 1, true, true, true, EPI_STORE_BF16)
    MOE_GEMM_CASE(256, 1, true, true, true, EPI_STORE_F32)
    MOE_GEMM_CASE(256, 1, false, false, false, EPI_STORE_BF16)
    MOE_GEMM_CASE(256, 1, false, false, false, EPI_STORE_F32)
    MOE_GEMM_CASE(256, 1, false, true, false, EPI_STORE_BF16)
    MOE_GEMM_CASE(256, 1, false, true, false, EPI_STORE_F32)
    MOE_GEMM_CASE(128, 2, false, false, false, EPI_STORE_BF16)  // 256 x 128 pair tiles (wave fit)
    MOE_GEMM_CASE(128, 2, false, false, false, EPI_STORE_F32)
    MOE_GEMM_CASE(128, 1, false, false, false, EPI_STORE_BF16)
    MOE_GEMM_CASE(128, 1, false, false, false, EPI_STORE_F32)
#undef MOE_GEMM_CASE
#undef MOE_GEMM_CASE_DISP
    return set_error(MOE_ERR_UNSUPPORTED,
                     "grouped GEMM variant not instantiated (bn=%d cg=%d a_mn=%d b_mn=%d kg=%d epi=%d)",
                     p.bn, p.cg, (int)p.a_mn, (int)p.b_mn, (int)p.k_grouped, p.epi);
}

// Tensor maps for the operand layouts used by the kernel.
moe_status tmap_kmajor(CUtensorMap* m, const void* base, int64_t rows, int64_t K, int box_rows) {
    return make_tmap_2d(m, base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (uint64_t)K, (uint64_t)rows,
                        (uint64_t)K * 2, 64, (uint32_t)box_rows);
}

moe_status tmap_mnmajor(CUtensorMap* m, const void* base, int64_t krows, int64_t mn) {
    return make_tmap_2d(m, base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (uint64_t)mn, (uint64_t)krows,
                        (uint64_t)mn * 2, 64, 64);
}

}  // namespace moe

using namespace moe;

extern "C" moe_status moe_grouped_gemm(const uint16_t* d_a, const uint16_t* d_b, void* d_d,
                                       int32_t groups, const int32_t* d_group_rows,
                                       int64_t total_rows, int64_t M, int64_t N, int64_t K,
                                       int32_t a_mn_major, int32_t b_mn_major,
                                       int32_t k_grouped, int32_t out_f32, int32_t bn,
                                       int32_t cta_pair, moe_stream_t stream) {
    const char* env = getenv("MOE_B_BOX_ROWS");
    const int b_box = env ? atoi(env) : 0;
    MOE_CHECK_ARG(d_a && d_b && d_d && d_group_rows, "null pointer");
    MOE_CHECK_ARG(bn == 128 || bn == 256, "bn must be 128 or 256");
    MOE_CHECK_ARG(N % 64 == 0 && K % 64 == 0 && M % 128 == 0 || !k_grouped, "K-grouped: M%128, N%64, K%64");
    MOE_CHECK_ARG(cta_pair == 0 || cta_pair == 1, "cta_pair must be 0 or 1");
    GemmPlan p;
    p.bn = bn;
    p.cg = cta_pair ? 2 : 1;
    p.a_mn = a_mn_major != 0;
    p.b_mn = b_mn_major != 0;
    p.k_grouped = k_grouped != 0;
    p.epi = out_f32 ? EPI_STORE_F32 : EPI_STORE_BF16;
    GemmArgs a{};
    a.G = groups;
    a.group_rows = d_group_rows;
    a.N = (int)N;
    a.out = d_d;
    a.ldo = N;
    if (!k_grouped) {
        // A [total_rows, K] K-major; B: K-major [G*N, K] or MN-major [G*K, N]
        MOE_CHECK_ARG(!a_mn_major, "M-grouped GEMM needs K-major A");
        MOE_CHECK_ARG(K % 8 == 0 && N % 8 == 0, "K and N must be multiples of 8");
        a.K = (int)K;
        MOE_TRY(tmap_kmajor(&p.ta, d_a, total_rows, K, 128));
        if (!b_mn_major) {
            a.b_group_stride = (int)N;
            a.b_box_rows = b_box > 0 ? b_box : bn / p.cg;   // = the CTA's B rows (256 / cg or 128 / cg)
            MOE_TRY(tmap_kmajor(&p.tb, d_b, (int64_t)groups * N, K, a.b_box_rows));
        } else {
            a.b_group_stride = (int)K;
            MOE_TRY(tmap_mnmajor(&p.tb, d_b, (int64_t)groups * K, N));
        }
    } else {
        // A [total_rows, M] MN-major, B [total_rows, N] MN-major, D [G*M, N]
        MOE_CHECK_ARG(a_mn_major && b_mn_major, "K-grouped GEMM needs MN-major A and B");
        a.K = (int)M;
        MOE_TRY(tmap_mnmajor(&p.ta, d_a, total_rows, M));
        MOE_TRY(tmap_mnmajor(&p.tb, d_b, total_rows, N));
    }
    return gemm_launch(p, a, (cudaStream_t)stream);
}

namespace {
__global__ void identity_rows_kernel(int32_t* v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (int32_t)i;
}
}  // namespace

/* The FP8 combine-payload epilogue (EPI_SCATTER_FP8) on its own: row r of the
 * grouped GEMM goes to row r of d_codes / d_scales (one destination rank). */
extern "C" moe_status moe_grouped_gemm_e4m3(const uint16_t* d_a, const uint16_t* d_b, uint8_t* d_codes,
                                            float* d_scales, int32_t groups, const int32_t* d_group_rows,
                                            int64_t total_rows, int64_t N, int64_t K, int32_t b_mn_major,
                                            int32_t cta_pair, moe_stream_t stream) {
    MOE_CHECK_ARG(d_a && d_b && d_codes && d_scales && d_group_rows, "null pointer");
    MOE_CHECK_ARG(N % 256 == 0 && K % 64 == 0, "N must be a multiple of 256, K of 64");
    MOE_CHECK_ARG(total_rows >= 0 && total_rows < (1ll << 27), "total_rows must be < 2^27");
    MOE_CHECK_ARG(cta_pair == 0 || cta_pair == 1, "cta_pair must be 0 or 1");
    cudaStream_t s = (cudaStream_t)stream;
    GemmPlan p;
    p.cg = cta_pair ? 2 : 1;
    p.b_mn = b_mn_major != 0;
    p.epi = EPI_SCATTER_FP8;
    MOE_TRY(tmap_kmajor(&p.ta, d_a, total_rows, K, 128));
    GemmArgs a{};
    a.G = groups;
    a.group_rows = d_group_rows;
    a.N = (int)N;
    a.K = (int)K;
    a.ldo = N;
    if (!p.b_mn) {
        a.b_group_stride = (int)N;
        MOE_TRY(tmap_kmajor(&p.tb, d_b, (int64_t)groups * N, K, 256 / p.cg));
    } else {
        a.b_group_stride = (int)K;
        MOE_TRY(tmap_mnmajor(&p.tb, d_b, (int64_t)groups * K, N));
    }
    // identity destinations on "rank 0" = the caller's buffers
    void* ws = nullptr;
    MOE_CUDA_TRY(cudaMallocAsync(&ws, 64 + (size_t)std::max<int64_t>(total_rows, 1) * 4, s));
    void* tables[2] = {d_codes, d_scales};
    MOE_CUDA_TRY(cudaMemcpyAsync(ws, tables, sizeof(tables), cudaMemcpyHostToDevice, s));
    int32_t* rows = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + 64);
    identity_rows_kernel<<<kNumSMs, 256, 0, s>>>(rows, total_rows);
    count_launch();
    a.row_dst = rows;
    a.rank_base = reinterpret_cast<void* const*>(ws);
    a.rank_scale_base = reinterpret_cast<void* const*>(ws) + 1;
    moe_status st = gemm_launch(p, a, s);
    cudaStreamSynchronize(s);  // the host table above must outlive the copy
    cudaFreeAsync(ws, s);
    return st;
}
