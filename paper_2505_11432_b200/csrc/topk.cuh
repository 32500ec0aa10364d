// topk.cuh — warp-level top-k over one token's router logits (ties -> lower
// expert id) and the softmax over the k picks (max-subtracted, fp32); shared by
// the routing kernels and the layer's fused router.
#pragma once

#include <cmath>
#include <cstdint>

namespace moe {

__device__ __forceinline__ void topk_select(const float* lg, int E, int k, int32_t* ex,
                                            float* gt, int lane) {
    // warp-parallel argmax rounds (k <= 8), ties -> lower expert id. For E <= 256
    // each lane keeps its (up to 8) logits in registers and a taken-mask; the
    // visiting order and comparisons are those of the generic loop below.
    float sel_val[8];
    int sel_id[8];
    const bool regs = E <= 256;
    float rv[8];
    unsigned taken_mask = 0;
    if (regs) {
#pragma unroll
        for (int q = 0; q < 8; ++q) rv[q] = (lane + 32 * q < E) ? lg[lane + 32 * q] : 0.0f;
    }
    for (int j = 0; j < k; ++j) {
        float best = -INFINITY;
        int bid = 0x7fffffff;
        if (regs) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int e = lane + 32 * q;
                if (e < E && !(taken_mask >> q & 1u)) {
                    const float v = rv[q];
                    if (v > best || (v == best && e < bid) || bid == 0x7fffffff) {
                        best = v;
                        bid = e;
                    }
                }
            }
        } else {
            for (int e = lane; e < E; e += 32) {
                bool taken = false;
                for (int i = 0; i < j; ++i) taken |= (sel_id[i] == e);
                const float v = lg[e];
                if (!taken && (v > best || (v == best && e < bid) || bid == 0x7fffffff)) {
                    best = v;
                    bid = e;
                }
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, best, off);
            const int oid = __shfl_xor_sync(0xffffffffu, bid, off);
            if (oid != 0x7fffffff && (bid == 0x7fffffff || ov > best || (ov == best && oid < bid))) {
                best = ov;
                bid = oid;
            }
        }
        sel_val[j] = best;
        sel_id[j] = bid;
        if (regs && bid != 0x7fffffff && (bid & 31) == lane) taken_mask |= 1u << (bid >> 5);
    }
    if (lane == 0) {
        // gates = softmax over the k selected logits (max-subtracted, fp32)
        const float m = sel_val[0];
        float s = 0.0f;
        float ev[8];
        for (int j = 0; j < k; ++j) {
            ev[j] = expf(sel_val[j] - m);
            s += ev[j];
        }
        for (int j = 0; j < k; ++j) {
            ex[j] = sel_id[j];
            gt[j] = ev[j] / s;
        }
    }
}

}  // namespace moe
