// runtime.cu — status plumbing, launch accounting, TMA descriptor encoding
// and the C-ABI entry points of the routing / quantisation operators.
#include <atomic>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include <cudaTypedefs.h>

#include "common.cuh"
#include "runtime.h"

namespace moe {

static thread_local char g_err[1024] = "";
static std::atomic<uint64_t> g_launches{0};

moe_status set_error(moe_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

moe_status make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt,
                        uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                        uint32_t box_outer, bool swizzle128) {
    auto fn = get_encode_fn();
    if (!fn) return set_error(MOE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return set_error(MOE_ERR_CUDA,
                         "cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu stride=%llu box=%u,%u",
                         (int)r, (unsigned long long)inner, (unsigned long long)outer,
                         (unsigned long long)row_bytes, box_inner, box_outer);
    return MOE_OK;
}

unsigned long long flag_timeout_ns() {
    static const unsigned long long ns = [] {
        const char* e = getenv("MOE_FLAG_TIMEOUT_MS");
        const long long ms = e ? atoll(e) : 0;
        return (unsigned long long)(ms > 0 ? ms : 20000) * 1000ull * 1000ull;
    }();
    return ns;
}

moe_status flag_status(const int* d_err, cudaStream_t s, const char* what) {
    MOE_CUDA_TRY(cudaStreamSynchronize(s));
    int v = 0;
    MOE_CUDA_TRY(cudaMemcpy(&v, d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (v == 0) return MOE_OK;
    if (v >= 8)
        return set_error(MOE_ERR_INTERNAL, "%s: debug-mode protocol assertion failed (code %d: %s)", what, v,
                         v == 8 ? "dispatch block arrivals != 128" : v == 9 ? "row claims did not reach the end"
                         : v == 10 ? "deduplicated row not landed exactly once" : v == 11 ? "all-gather chunk incomplete"
                         : "barrier epoch mismatch (16 + slot)");
    static const char* kinds[] = {"", "cross-GPU flag barrier", "fused-dispatch row arrival",
                                  "DP in-place cast chunk", "GEMM-RS tile arrival"};
    return set_error(MOE_ERR_TIMEOUT, "%s: a %s wait exceeded its bound (a peer rank stalled or "
                     "failed); results of the affected calls are invalid", what,
                     (v >= 1 && v <= 4) ? kinds[v] : "device");
}

}  // namespace moe

using namespace moe;

extern "C" {

const char* moe_last_error(void) { return g_err; }
int moe_version(void) { return 1; }
uint64_t moe_launch_count(void) { return g_launches.load(); }
void moe_launch_count_reset(void) { g_launches.store(0); }

moe_status moe_capacity_drop(const int32_t* d_experts, int64_t T, int64_t E, int64_t k,
                             int64_t n_groups, double capacity_factor, uint8_t* d_dropped,
                             moe_stream_t stream) {
    return launch_capacity_drop(d_experts, T, E, k, n_groups, capacity_factor, d_dropped,
                                (cudaStream_t)stream);
}

size_t moe_permute_workspace_size(int64_t T, int64_t E, int64_t k, int64_t n_src) {
    return permute_workspace_bytes(T, E, k, n_src);
}

moe_status moe_permute(const int32_t* d_experts, const int32_t* d_source_rank,
                       const uint8_t* d_dropped, int64_t T, int64_t E, int64_t k, int64_t n,
                       int64_t my_rank, int64_t n_src, int32_t* d_row_map_in,
                       int32_t* d_per_expert_counts, int32_t* d_out_expert,
                       int32_t* d_out_source_rank, int32_t* d_expert_offsets, int32_t* d_rows,
                       void* d_workspace, moe_stream_t stream) {
    return launch_permute(d_experts, d_source_rank, d_dropped, T, E, k, n, my_rank, n_src,
                          d_row_map_in, d_per_expert_counts, d_out_expert, d_out_source_rank,
                          d_expert_offsets, d_rows, d_workspace, nullptr, nullptr, nullptr, 128,
                          (cudaStream_t)stream);
}

moe_status moe_tile_layout(const int32_t* d_out_source_rank, const int32_t* d_expert_offsets,
                           int64_t num_local_experts, int64_t first_expert, int64_t tile_rows,
                           int32_t* d_tile_expert, int32_t* d_tile_begin, int32_t* d_tile_end,
                           uint64_t* d_tile_rank_mask, int32_t* d_num_tiles,
                           moe_stream_t stream) {
    return launch_tile_layout(d_out_source_rank, d_expert_offsets, num_local_experts, first_expert,
                              tile_rows, d_tile_expert, d_tile_begin, d_tile_end,
                              d_tile_rank_mask, d_num_tiles, (cudaStream_t)stream);
}

moe_status moe_balance_counts(const int32_t* d_experts, const uint8_t* d_dropped, int64_t T,
                              int64_t E, int64_t k, int64_t n, int64_t* d_per_group_load,
                              int64_t* d_assigned, int64_t* d_dropped_tokens,
                              moe_stream_t stream) {
    return launch_balance_counts(d_experts, d_dropped, T, E, k, n, d_per_group_load, d_assigned,
                                 d_dropped_tokens, (cudaStream_t)stream);
}

moe_status moe_router_topk(const uint16_t* d_x, const uint16_t* d_wr, int64_t T, int64_t h,
                           int64_t E, int64_t k, float* d_logits, int32_t* d_experts,
                           float* d_gates, moe_stream_t stream) {
    return launch_router_topk(d_x, d_wr, T, h, E, k, d_logits, d_experts, d_gates,
                              (cudaStream_t)stream);
}

moe_status moe_topk_from_logits(const float* d_logits, int64_t T, int64_t E, int64_t k,
                                int32_t* d_experts, float* d_gates, moe_stream_t stream) {
    return launch_topk_from_logits(d_logits, T, E, k, d_experts, d_gates, (cudaStream_t)stream);
}

moe_status moe_quantize_e4m3_rows(const uint16_t* d_x, int64_t rows, int64_t cols,
                                  uint8_t* d_codes, float* d_scales, moe_stream_t stream) {
    return launch_quantize_e4m3_rows(d_x, false, rows, cols, d_codes, d_scales,
                                     (cudaStream_t)stream);
}

moe_status moe_quantize_e4m3_rows_f32(const float* d_x, int64_t rows, int64_t cols,
                                      uint8_t* d_codes, float* d_scales, moe_stream_t stream) {
    return launch_quantize_e4m3_rows(d_x, true, rows, cols, d_codes, d_scales,
                                     (cudaStream_t)stream);
}

}  // extern "C"
