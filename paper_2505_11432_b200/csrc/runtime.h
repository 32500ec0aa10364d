// runtime.h — host-side internals shared by the translation units of
// libmoe_b200.so: launch accounting, TMA descriptor encoding, kernel
// launchers. Not part of the public C ABI (that is include/moe_b200.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/moe_b200.h"

namespace moe {

void count_launch(int n = 1);

// 2-D bf16/fp32/u8 tensor map, 128B swizzle, box {box_inner, box_outer}.
// inner = contiguous dimension (elements), outer = rows; row_bytes = stride.
moe_status make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dt,
                        uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                        uint32_t box_outer, bool swizzle128 = true);

// ---- routing.cu ----
moe_status launch_router_topk(const uint16_t* x, const uint16_t* wr, int64_t T, int64_t h,
                              int64_t E, int64_t k, float* logits, int32_t* experts, float* gates,
                              cudaStream_t s);
moe_status launch_topk_from_logits(const float* logits, int64_t T, int64_t E, int64_t k,
                                   int32_t* experts, float* gates, cudaStream_t s);
moe_status launch_capacity_drop(const int32_t* experts, int64_t T, int64_t E, int64_t k,
                                int64_t n_groups, double cf, uint8_t* dropped, cudaStream_t s);
size_t permute_workspace_bytes(int64_t T, int64_t E, int64_t k, int64_t n_src);
moe_status launch_permute(const int32_t* experts, const int32_t* src, const uint8_t* dropped,
                          int64_t T, int64_t E, int64_t k, int64_t n, int64_t my_rank,
                          int64_t n_src, int32_t* row_map_in, int32_t* per_expert_counts,
                          int32_t* out_expert, int32_t* out_src, int32_t* expert_offsets,
                          int32_t* rows, void* workspace, int32_t* group_pad_rows,
                          int32_t* group_pad_off, int32_t* pad_row_tok, int pad,
                          cudaStream_t s);
moe_status launch_tile_layout(const int32_t* out_src, const int32_t* expert_offsets, int64_t el,
                              int64_t first, int64_t tile_rows, int32_t* t_expert,
                              int32_t* t_begin, int32_t* t_end, uint64_t* t_mask,
                              int32_t* n_tiles, cudaStream_t s);
moe_status launch_balance_counts(const int32_t* experts, const uint8_t* dropped, int64_t T,
                                 int64_t E, int64_t k, int64_t n, int64_t* load,
                                 int64_t* assigned, int64_t* ndrop, cudaStream_t s);

// Bound of a cross-GPU flag barrier wait before it gives up and sets the
// error flag (MOE_FLAG_TIMEOUT_MS, default 20000 ms; read once).
unsigned long long flag_timeout_ns();

// Device error flag of a handle -> status: synchronises `s`, then returns
// MOE_ERR_TIMEOUT when a bounded cross-GPU wait gave up (1 = flag barrier,
// 2 = fused-dispatch row wait, 3 = DP in-place cast wait).
moe_status flag_status(const int* d_err, cudaStream_t s, const char* what);

// ---- quant.cu ----
moe_status launch_quantize_e4m3_rows(const void* x, bool x_is_f32, int64_t rows, int64_t cols,
                                     uint8_t* codes, float* scales, cudaStream_t s);

}  // namespace moe
