// gemm.h — host-side plan for the tcgen05 grouped GEMM.
#pragma once

#include "gemm_sm100.cuh"
#include "runtime.h"

namespace moe {

struct GemmPlan {
    CUtensorMap ta, tb;
    int bn = 256;
    int cg = 1;       // 2 = CTA pair (cta_group::2, 256-row tiles)
    bool a_mn = false, b_mn = false, k_grouped = false;
    int epi = EPI_STORE_BF16;
    bool dispatch = false;  // fused AG + scatter of the A operand
    int grid = 0;  // 0 = one CTA per SM
    // dynamic-schedule tile counter owned by the plan's object (layer, attn,
    // ulysses), so a CUDA graph that captured it never shares it with a later
    // eager launch; nullptr = the stateless operators' per-device ring
    int* counter = nullptr;
};

moe_status gemm_launch(const GemmPlan& p, const GemmArgs& a, cudaStream_t s);
moe_status tmap_kmajor(CUtensorMap* m, const void* base, int64_t rows, int64_t K, int box_rows);
moe_status tmap_mnmajor(CUtensorMap* m, const void* base, int64_t krows, int64_t mn);

}  // namespace moe

