// layer.cu — the MoE layer handle: router -> dispatch (AG + local scatter)
// -> fc1 GroupedGEMM + SwiGLU (+ gate) -> fc2 GroupedGEMM + gather to the
// source rank -> combine, and the mirrored backward with the paper's
// selective rematerialisation of fc2_in from the retained fc1_out
// (graph.cpp:254-311 forward, :333-401 backward).
//
// Multi-GPU (ep_size = n > 1): one process per GPU. Every rank owns one
// symmetric arena (identical offsets on every rank) exported with CUDA IPC;
// peers' arenas are mapped over NVLink. Dispatch pulls token rows straight
// from the owning rank's input buffer into permuted order inside the fc1 /
// fc2-dgrad GEMM (fused AG + scatter); the fc2 / fc1-dgrad epilogues store
// each output row into the owning rank's combine staging (fused gather +
// RS); device flag barriers (st.release.sys / ld.acquire.sys) separate the
// phases. FP8 communication sends E4M3 codes + fp32
// scales on all four exchanges: per-token for the forward dispatch,
// grouped-128 for the combine payloads and the backward dispatch.
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gemm.h"
#include "layer_kernels.cuh"
#include "runtime.h"

namespace moe {

namespace {
size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

// fields of the symmetric arena (same offsets on every rank)
enum Field {
    F_X, F_DY, F_STAGE, F_DSTAGE, F_EX, F_GT, F_DGATE, F_FLAGS,
    F_X8, F_XSC, F_DY8, F_DYSC, F_STAGE8, F_SSC, F_DSTAGE8, F_DSSC,
    F_RSTAGE,  // ag_rs: reduce-scatter staging [T_r, n, h] (one partial per serving rank)
    F_COUNT
};
}  // namespace

constexpr int kStampSlots = 64;  // PH_COUNT phase stamps + 2 per barrier slot (4 slots)

enum Phase {
    PH_ROUTE, PH_PERMUTE, PH_DISPATCH, PH_FC1, PH_FC2, PH_COMBINE, PH_FWD_END,
    PH_DISPATCH_DY, PH_FC2_DGRAD, PH_FC1_DGRAD, PH_DGATE, PH_COMBINE_DX, PH_FC2_WGRAD,
    PH_FC1_WGRAD, PH_ROUTER_WGRAD, PH_END, PH_COUNT
};
static const char* kPhaseNames[PH_COUNT] = {
    "route", "permute", "dispatch", "fc1", "fc2", "combine", "fwd_end", "dispatch_dy", "fc2_dgrad",
    "fc1_dgrad", "dgate", "combine_dx", "fc2_wgrad", "fc1_wgrad", "router_wgrad", "end"};

}  // namespace moe

struct moe_layer {
    moe_layer_config cfg{};
    int64_t Tr = 0, T = 0, h = 0, f = 0, E = 0, k = 0, n = 1, rank = 0, el = 0, first = 0, Mp = 0;
    int dev = 0;
    bool fp8 = false, gate_after = false;
    // GEMM tiling: cg = 2 -> CTA-pair 256-row tiles (a segment's odd 128-row
    // block as an M = 128 pair tile); cg = 1 -> 128-row tiles for fine-grained
    // experts. Expert segments are padded to 128 rows either way.
    int cg = 2, pad = 128;
    bool norm = false;         // ffn_norm fused ahead of router / dispatch
    uint16_t* x_res = nullptr;  // pre-norm input [T_r, h]
    uint16_t* dxn = nullptr;    // d(normed input) [T_r, h]
    float *gamma = nullptr, *rstd = nullptr, *dgamma = nullptr, *dgamma_part = nullptr;
    bool gemm_router = false;  // router logits on the tensor cores (large E*h)
    bool gemm_router_wgrad = false;  // dWr = dlogits^T x on the tensor cores (E >= 128)
    uint16_t* dlogits_bf16 = nullptr;
    moe::GemmPlan p_router_wgrad;
    int32_t* router_rows = nullptr;
    moe::GemmPlan p_router;
    // symmetric arena (IPC-exported)
    uint8_t* arena = nullptr;
    size_t arena_bytes = 0;
    size_t off[moe::F_COUNT] = {};
    std::vector<uint8_t*> peer_arena;  // [n], self included
    // per-field pointer tables [F_COUNT][n]: remote (peers' arenas) and
    // local (every entry = this rank: compute-only measurement mode)
    void** tab_remote = nullptr;
    void** tab_local = nullptr;
    bool comm_local = false;
    // local buffers
    uint16_t *w1p = nullptr, *w2 = nullptr, *wr = nullptr;
    int32_t* ex_loc = nullptr;
    float *gt_loc = nullptr, *logits = nullptr;
    int32_t* src = nullptr;
    uint8_t* dropped = nullptr;
    void* perm_ws = nullptr;
    int32_t *row_map_in = nullptr, *out_expert = nullptr, *out_src = nullptr, *counts = nullptr,
            *expert_off = nullptr, *rows = nullptr, *gpad_rows = nullptr, *gpad_off = nullptr,
            *pad_tok = nullptr, *row_dst = nullptr;
    float* row_gate = nullptr;
    uint16_t *x_perm = nullptr, *fc1_out = nullptr, *fc2_in = nullptr, *dy_perm = nullptr,
             *dfc1 = nullptr;
    float *dgate_part = nullptr, *dlogits = nullptr, *rw_part = nullptr;
    uint32_t* ready = nullptr;  // fused-dispatch arrival counters [Mp / L->pad]
    // dispatch dedup when a token has several experts on this rank (k > 1,
    // E/n > 1): later rows copy the first landed row instead of re-pulling it
    bool dedup = false;
    int32_t *first_row = nullptr, *dup_src = nullptr;
    uint32_t* row_done = nullptr;
    bool fused_dispatch = true;
    // ep_pattern = ag_rs (n > 1): in-kernel all-gather of every peer's rows into
    // x_all, local scatter from it; expert outputs stored locally, pre-reduced
    // per (token, rank) and reduce-scattered to the owner
    bool ag = false;
    // MOE_DEBUG_CHECKS=1: device-side protocol assertions (barrier epochs, dispatch
    // arrivals) that set the error flag; moe_layer_status reports them
    bool debug = false;
    uint16_t* x_all = nullptr;      // [T, h] (x in forward, dy in backward)
    uint32_t* ag_ready = nullptr;   // [n][ceil(T_r/64)] rows landed per 64-token chunk
    int32_t* inv = nullptr;         // [T*k] padded row of (t, slot), -1 = not here
    uint16_t* rows_out = nullptr;   // [Mp, h] local fc2 / fc1-dgrad output rows
    moe::GemmPlan p_fc2_local, p_fc1_dgrad_local;
    int* err = nullptr;
    int* err_host = nullptr;  // pinned mirror of *err, refreshed at the end of multi-GPU calls
    uint32_t* epoch_dev = nullptr;
    int* counters = nullptr;  // dynamic tile schedule counters, one per GEMM plan
    // E <= 8 router: h split over router_split CTAs per 16-token block
    int router_split = 1;
    float* router_part = nullptr;
    unsigned* router_cnt = nullptr;
    bool router_attr = false;
    bool weights_set = false, routing_set = false, fwd_done = false, ipc_ready = false;
    int stage = 0;  // forward stages done: 1 = routed, 2 = dispatch + fc1
    // GEMM plans (tensor maps fixed at create)
    moe::GemmPlan p_fc1, p_fc2, p_fc2_dgrad, p_fc2_wgrad, p_fc1_dgrad, p_fc1_wgrad;
    // timing
    bool timing = false;
    cudaEvent_t ev[moe::PH_COUNT] = {};
    bool ev_used[moe::PH_COUNT] = {};

    template <class T>
    T* mine(int field) { return reinterpret_cast<T*>(arena + off[field]); }
    // device array of n per-rank pointers for `field`
    template <class T>
    T* const* tab(int field) const {
        return reinterpret_cast<T* const*>((comm_local ? tab_local : tab_remote) + field * n);
    }
    // %globaltimer trace: stamps[ph] at each phase boundary, stamps[PH_COUNT +
    // 2*slot + {0,1}] at each barrier's entry / release (captured into graphs)
    bool stamping = false;
    unsigned long long* stamps = nullptr;
    void mark(int ph, cudaStream_t s) {
        if (timing) {
            cudaEventRecord(ev[ph], s);
            ev_used[ph] = true;
        }
        if (stamping) {
            moe::stamp_kernel<<<1, 32, 0, s>>>(stamps + ph);
            moe::count_launch();
        }
    }
};

using namespace moe;

namespace {

template <class T>
moe_status dalloc(T** p, size_t count) {
    MOE_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T)));
    return MOE_OK;
}

moe_status fill_tables(moe_layer* L) {
    const int n = (int)L->n;
    std::vector<void*> remote(F_COUNT * n), local(F_COUNT * n);
    for (int fld = 0; fld < F_COUNT; ++fld)
        for (int p = 0; p < n; ++p) {
            remote[fld * n + p] = L->peer_arena[p] + L->off[fld];
            local[fld * n + p] = L->arena + L->off[fld];
        }
    MOE_CUDA_TRY(cudaMemcpy(L->tab_remote, remote.data(), sizeof(void*) * remote.size(), cudaMemcpyHostToDevice));
    MOE_CUDA_TRY(cudaMemcpy(L->tab_local, local.data(), sizeof(void*) * local.size(), cudaMemcpyHostToDevice));
    return MOE_OK;
}

moe_status build_plans(moe_layer* L) {
    const int64_t Mp = L->Mp, h = L->h, f = L->f, el = L->el;
    // forward fc1: A = x_perm [Mp, h], B = w1p [el*2f, h] (K-major)
    L->p_fc1 = GemmPlan{};
    L->p_fc1.epi = EPI_SWIGLU;
    MOE_TRY(tmap_kmajor(&L->p_fc1.ta, L->x_perm, Mp, h, 128));
    MOE_TRY(tmap_kmajor(&L->p_fc1.tb, L->w1p, el * 2 * f, h, 256 / L->cg));
    // forward fc2: A = fc2_in [Mp, f], B = w2 [el*h, f] (K-major)
    L->p_fc2 = GemmPlan{};
    L->p_fc2.epi = L->fp8 ? EPI_SCATTER_FP8 : EPI_SCATTER;
    MOE_TRY(tmap_kmajor(&L->p_fc2.ta, L->fc2_in, Mp, f, 128));
    MOE_TRY(tmap_kmajor(&L->p_fc2.tb, L->w2, el * h, f, 256 / L->cg));
    // fc2 dgrad: A = dy_perm [Mp, h], B(n=f, k=h) = w2[e][k][n] (MN-major)
    L->p_fc2_dgrad = GemmPlan{};
    L->p_fc2_dgrad.epi = EPI_SWIGLU_BWD;
    L->p_fc2_dgrad.b_mn = true;
    MOE_TRY(tmap_kmajor(&L->p_fc2_dgrad.ta, L->dy_perm, Mp, h, 128));
    MOE_TRY(tmap_mnmajor(&L->p_fc2_dgrad.tb, L->w2, el * h, f));
    // fc2 wgrad: dW2[e] = dy_perm^T fc2_in (K-grouped, MN-major both)
    L->p_fc2_wgrad = GemmPlan{};
    L->p_fc2_wgrad.epi = EPI_STORE_BF16;
    L->p_fc2_wgrad.a_mn = L->p_fc2_wgrad.b_mn = L->p_fc2_wgrad.k_grouped = true;
    MOE_TRY(tmap_mnmajor(&L->p_fc2_wgrad.ta, L->dy_perm, Mp, h));
    MOE_TRY(tmap_mnmajor(&L->p_fc2_wgrad.tb, L->fc2_in, Mp, f));
    // fc1 dgrad: A = dfc1 [Mp, 2f], B(n=h, k=j) = w1p[e][j][n] (MN-major)
    L->p_fc1_dgrad = GemmPlan{};
    L->p_fc1_dgrad.epi = L->fp8 ? EPI_SCATTER_FP8 : EPI_SCATTER;
    L->p_fc1_dgrad.b_mn = true;
    MOE_TRY(tmap_kmajor(&L->p_fc1_dgrad.ta, L->dfc1, Mp, 2 * f, 128));
    MOE_TRY(tmap_mnmajor(&L->p_fc1_dgrad.tb, L->w1p, el * 2 * f, h));
    // fc1 wgrad: dW1p[e] = dfc1^T x_perm (K-grouped)
    L->p_fc1_wgrad = GemmPlan{};
    L->p_fc1_wgrad.epi = EPI_STORE_BF16;
    L->p_fc1_wgrad.a_mn = L->p_fc1_wgrad.b_mn = L->p_fc1_wgrad.k_grouped = true;
    MOE_TRY(tmap_mnmajor(&L->p_fc1_wgrad.ta, L->dfc1, Mp, 2 * f));
    MOE_TRY(tmap_mnmajor(&L->p_fc1_wgrad.tb, L->x_perm, Mp, h));
    int ci = 0;
    for (GemmPlan* p : {&L->p_fc1, &L->p_fc2, &L->p_fc2_dgrad, &L->p_fc2_wgrad, &L->p_fc1_dgrad,
                        &L->p_fc1_wgrad}) {
        p->cg = L->cg;
        p->counter = L->counters + ci++;
    }
    // ag_rs: the same GEMMs with a plain local row-major store epilogue
    L->p_fc2_local = L->p_fc2;
    L->p_fc2_local.epi = EPI_STORE_BF16;
    L->p_fc2_local.counter = L->counters + 8;
    L->p_fc1_dgrad_local = L->p_fc1_dgrad;
    L->p_fc1_dgrad_local.epi = EPI_STORE_BF16;
    L->p_fc1_dgrad_local.counter = L->counters + 9;
    // router logits[T_r, E] = x . wr^T on the tensor cores when W_r does not
    // fit in shared memory (DeepSeek shape: E = 256, h = 7168)
    L->gemm_router = (size_t)L->E * h * 4 > 200 * 1024 || L->E > 64;
    if (L->gemm_router) {
        L->p_router = GemmPlan{};
        L->p_router.epi = EPI_STORE_F32;
        L->p_router.counter = L->counters + 6;
        // only T_r/128 x E/128 output tiles: single-CTA 128 x 128 tiles keep
        // 4x more SMs busy than 256 x 256 pairs (E = 256: 49 -> ~20 us)
        L->p_router.bn = 128;
        L->p_router.cg = 1;
        MOE_TRY(tmap_kmajor(&L->p_router.ta, L->arena + L->off[F_X], L->Tr, h, 128));
        MOE_TRY(tmap_kmajor(&L->p_router.tb, L->wr, L->E, h, 128));
        const int32_t rr = (int32_t)L->Tr;
        MOE_CUDA_TRY(cudaMemcpy(L->router_rows, &rr, sizeof(rr), cudaMemcpyHostToDevice));
    }
    // router weight gradient as a K-grouped GEMM (rows = tokens) when E is a
    // multiple of the tile height: dWr[E, h] = dlogits[T_r, E]^T . x[T_r, h]
    L->gemm_router_wgrad = L->E % 256 == 0 && L->Tr % 64 == 0;
    if (L->gemm_router_wgrad) {
        L->p_router_wgrad = GemmPlan{};
        L->p_router_wgrad.epi = EPI_STORE_F32;
        L->p_router_wgrad.counter = L->counters + 7;
        L->p_router_wgrad.cg = 2;
        L->p_router_wgrad.a_mn = L->p_router_wgrad.b_mn = L->p_router_wgrad.k_grouped = true;
        MOE_TRY(tmap_mnmajor(&L->p_router_wgrad.ta, L->dlogits_bf16, L->Tr, L->E));
        MOE_TRY(tmap_mnmajor(&L->p_router_wgrad.tb, L->arena + L->off[F_X], L->Tr, h));
        const int32_t rr = (int32_t)L->Tr;
        MOE_CUDA_TRY(cudaMemcpy(L->router_rows, &rr, sizeof(rr), cudaMemcpyHostToDevice));
    }
    return MOE_OK;
}

// Fused dispatch (AG + local scatter) of one of the two pulled operands.
void set_dispatch(moe_layer* L, GemmArgs& a, bool backward, uint16_t* dst) {
    // with peers to pull from, the first wave should need only the first 8
    // row blocks; on one GPU the whole-group raster reads each weight once
    // (also in compute-only mode, so that mode runs the identical tile order)
    if (L->fused_dispatch && L->n > 1) a.m_chunk = 8;
    a.pad_row_tok = L->pad_tok;
    a.nrows_pad = L->gpad_off + L->el;
    a.a_dst = dst;
    a.ready = L->ready;
    a.row_claim = reinterpret_cast<int*>(L->ready + L->Mp / L->pad + 1);
    a.topk = (int)L->k;
    a.tokens_per_rank = (int)L->Tr;
    a.err = L->err;
    if (L->ag) {
        a.ag_rows = (int)((L->n - 1) * L->Tr);
        a.self_rank = (int)L->rank;
        a.ag_dst = L->x_all;
        a.ag_ready = L->ag_ready;
        a.n_src = (int)L->n;
    }
    // the backward copy would carry the first row's gate (gate after fc2): pull instead
    if (L->dedup && !(backward && L->gate_after)) {
        a.dup_src = L->dup_src;
        a.row_done = L->row_done;
    }
    if (!backward) {
        a.src_bufs = L->tab<const uint16_t>(F_X);
        if (L->fp8) {
            a.src_bufs8 = L->tab<const uint8_t>(F_X8);
            a.src_scales = L->tab<const float>(F_XSC);
            a.src_scale_group = (int)L->h;  // per-token
        }
    } else {
        a.src_bufs = L->tab<const uint16_t>(F_DY);
        if (L->fp8) {
            a.src_bufs8 = L->tab<const uint8_t>(F_DY8);
            a.src_scales = L->tab<const float>(F_DYSC);
            a.src_scale_group = 128;        // grouped-128 in backward
        }
        // gate after fc2: d fc2_out = gate * dy
        if (L->gate_after) a.row_scale = L->row_gate;
    }
}

moe_status barrier(moe_layer* L, int slot, cudaStream_t s, int bump) {
    if (L->n == 1 || L->comm_local) return MOE_OK;
    if (!L->ipc_ready) return set_error(MOE_ERR_INVALID, "ep_size > 1 requires moe_layer_ipc_import");
    flag_barrier_kernel<<<1, 64, 0, s>>>(L->tab<uint32_t>(F_FLAGS), slot, (int)L->n, (int)L->rank,
                                        L->epoch_dev, bump, flag_timeout_ns(), L->err,
                                        L->stamping ? L->stamps + PH_COUNT + 2 * slot : nullptr, (int)L->debug);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

// debug mode: the fused-dispatch protocol invariants after a fused GEMM
moe_status debug_check_dispatch(moe_layer* L, bool backward, cudaStream_t s) {
    if (!L->debug || !L->fused_dispatch) return MOE_OK;
    const bool dd = L->dedup && !(backward && L->gate_after);
    dispatch_check_kernel<<<kNumSMs, 256, 0, s>>>(
        L->ready, (int)(L->Mp / L->pad + 1), L->gpad_off + L->el,
        reinterpret_cast<const int*>(L->ready + L->Mp / L->pad + 1), L->ag ? (int)((L->n - 1) * L->Tr) : 0,
        dd ? L->row_done : nullptr, L->pad_tok, L->ag ? L->ag_ready : nullptr, (int)L->n, (int)L->rank,
        (int)L->Tr, L->err);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

// ag_rs gather + reduce-scatter: per (token, this rank) partial of the local
// slot rows -> the owning rank's F_RSTAGE[t_local][rank].
moe_status launch_gather_rs(moe_layer* L, cudaStream_t s) {
    gather_rs_kernel<<<kNumSMs * 4, 256, 0, s>>>(L->mine<int32_t>(F_EX), L->dropped, L->inv, (int)L->T, (int)L->k,
                                                 (int)L->first, (int)L->el, (int)L->Tr, (int)L->n, (int)L->rank,
                                                 (int)L->h, L->rows_out, L->tab<uint16_t>(F_RSTAGE));
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

// A timeout of an earlier call that has reached the host (non-blocking).
moe_status pending_timeout(moe_layer* L) {
    const int v = *reinterpret_cast<volatile int*>(L->err_host);
    if (v == 0) return MOE_OK;
    if (v >= 8) return set_error(MOE_ERR_INTERNAL, "moe_layer: debug-mode protocol assertion %d in an earlier call", v);
    return set_error(MOE_ERR_TIMEOUT, "moe_layer: an earlier call's cross-GPU wait timed out (kind %d); "
                     "its results are invalid (moe_layer_clear_error resets)", v);
}

// Mirror the device flag into pinned host memory at the end of a multi-GPU
// call (one 4-byte copy; graph-capturable).
moe_status mirror_error(moe_layer* L, cudaStream_t s) {
    if (L->n == 1 || L->comm_local) return MOE_OK;
    MOE_CUDA_TRY(cudaMemcpyAsync(L->err_host, L->err, sizeof(int), cudaMemcpyDeviceToHost, s));
    return MOE_OK;
}

moe_status quantize_rows(const uint16_t* x, int64_t rows, int64_t cols, bool per_token,
                         uint8_t* codes, float* scales, cudaStream_t s) {
    const int grid = (int)std::min<int64_t>((rows + 7) / 8, kNumSMs * 8);
    if (per_token)
        quantize_fast_kernel<0><<<grid, 256, 0, s>>>(x, (int)rows, (int)cols, codes, scales);
    else
        quantize_fast_kernel<128><<<grid, 256, 0, s>>>(x, (int)rows, (int)cols, codes, scales);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

}  // namespace

extern "C" {

moe_status moe_layer_create(const moe_layer_config* cfg, moe_layer** out) {
    MOE_CHECK_ARG(cfg && out, "null argument");
    const moe_layer_config c = *cfg;
    MOE_CHECK_ARG(c.tokens_per_rank >= 1 && c.hidden >= 256 && c.ffn_hidden >= 256,
                  "tokens_per_rank >= 1, hidden and ffn_hidden >= 256");
    MOE_CHECK_ARG(c.hidden % 256 == 0, "hidden must be a multiple of 256");
    MOE_CHECK_ARG(c.ffn_hidden % 256 == 0, "ffn_hidden must be a multiple of 256");
    MOE_CHECK_ARG(c.num_experts >= 1 && c.top_k >= 1 && c.top_k <= 8 && c.top_k <= c.num_experts,
                  "need 1 <= top_k <= min(8, num_experts)");
    // row destinations pack the source rank as (rank << 27) | row into a signed
    // int32 (negative = padding row), so ranks 0..15 round-trip
    MOE_CHECK_ARG(c.ep_size >= 1 && c.ep_size <= 16 && c.num_experts % c.ep_size == 0,
                  "num_experts must be divisible by ep_size (<= 16)");
    MOE_CHECK_ARG(c.rank >= 0 && c.rank < c.ep_size, "rank out of range");
    MOE_CHECK_ARG(c.num_experts / c.ep_size <= 256, "at most 256 local experts");
    MOE_CHECK_ARG(c.comm_format == MOE_COMM_BF16 || c.comm_format == MOE_COMM_FP8,
                  "comm_format must be bf16 or fp8");
    MOE_CHECK_ARG(c.gate_order == MOE_GATE_BEFORE_FC2 || c.gate_order == MOE_GATE_AFTER_FC2,
                  "gate_order must be before_fc2_in or after_fc2_out");
    MOE_CHECK_ARG(c.ep_pattern == MOE_EP_A2A || c.ep_pattern == MOE_EP_AG_RS, "ep_pattern must be a2a or ag_rs");
    if (c.ep_pattern == MOE_EP_AG_RS && c.ep_size > 1 &&
        (c.comm_format != MOE_COMM_BF16 || c.gate_order != MOE_GATE_BEFORE_FC2))
        return set_error(MOE_ERR_UNSUPPORTED,
                         "ep_pattern ag_rs is built for bf16 communication with the gate before fc2 "
                         "(the FP8 / gate-after-fc2 path uses a2a)");
    auto* L = new moe_layer();
    L->cfg = c;
    L->fp8 = c.comm_format == MOE_COMM_FP8;
    L->gate_after = c.gate_order == MOE_GATE_AFTER_FC2;
    L->ag = c.ep_pattern == MOE_EP_AG_RS && c.ep_size > 1;
    L->Tr = c.tokens_per_rank;
    L->n = c.ep_size;
    L->rank = c.rank;
    L->T = L->Tr * L->n;
    L->h = c.hidden;
    L->f = c.ffn_hidden;
    L->E = c.num_experts;
    L->k = c.top_k;
    L->el = L->E / L->n;
    L->first = L->rank * L->el;
    {
        // CTA pairs are 13-22% faster per FLOP at these shapes
        // (scripts/perf_gemm_deepseek.py); padding to 256 instead of 128 rows
        // costs ~64 more rows per expert on average: pairs win above ~256 rows/expert
        const double rows_per_expert = double(L->T * L->k) / double(L->E);
        L->cg = rows_per_expert >= 256.0 ? 2 : 1;
        if (const char* e = getenv("MOE_GEMM_CG")) L->cg = atoi(e) == 1 ? 1 : 2;
        L->pad = 128;   // CTA pairs run a group's odd 128-row block as an M = 128 pair tile
    }
    L->Mp = L->T * L->k + L->el * L->pad;
    MOE_CHECK_ARG(L->T * L->k < (1ll << 27), "T*k must be < 2^27");
    cudaGetDevice(&L->dev);

    // ---- symmetric arena ----
    const int64_t Tr = L->Tr, h = L->h, k = L->k;
    size_t sizes[F_COUNT] = {};
    sizes[F_X] = Tr * h * 2;
    sizes[F_DY] = Tr * h * 2;
    sizes[F_STAGE] = Tr * k * h * 2;
    sizes[F_DSTAGE] = Tr * k * h * 2;
    sizes[F_EX] = L->T * k * 4;
    sizes[F_GT] = L->T * k * 4;
    sizes[F_DGATE] = Tr * k * 4;
    sizes[F_FLAGS] = 16 * 64 * 4;
    sizes[F_X8] = L->fp8 ? Tr * h : 0;
    sizes[F_XSC] = L->fp8 ? Tr * 4 : 0;
    sizes[F_DY8] = L->fp8 ? Tr * h : 0;
    sizes[F_DYSC] = L->fp8 ? Tr * (h / 128) * 4 : 0;
    sizes[F_STAGE8] = L->fp8 ? Tr * k * h : 0;
    sizes[F_SSC] = L->fp8 ? Tr * k * (h / 128) * 4 : 0;
    sizes[F_DSTAGE8] = L->fp8 ? Tr * k * h : 0;
    sizes[F_DSSC] = L->fp8 ? Tr * k * (h / 128) * 4 : 0;
    sizes[F_RSTAGE] = L->ag ? Tr * L->n * h * 2 : 0;
    size_t total = 0;
    for (int fld = 0; fld < F_COUNT; ++fld) {
        L->off[fld] = total;
        total = align_up(total + sizes[fld]);
    }
    L->arena_bytes = total;
    moe_status st = MOE_OK;
#define TRY_ALLOC(expr) do { st = (expr); if (st != MOE_OK) { moe_layer_destroy(L); return st; } } while (0)
    TRY_ALLOC(dalloc(&L->arena, L->arena_bytes));
    cudaMemset(L->arena, 0, L->arena_bytes);
    L->peer_arena.assign(L->n, nullptr);
    L->peer_arena[L->rank] = L->arena;
    const int64_t Mp = L->Mp, f = L->f, el = L->el;
    TRY_ALLOC(dalloc(&L->w1p, el * 2 * f * h));
    TRY_ALLOC(dalloc(&L->w2, el * h * f));
    TRY_ALLOC(dalloc(&L->wr, L->E * h));
    TRY_ALLOC(dalloc(&L->ex_loc, Tr * k));
    TRY_ALLOC(dalloc(&L->gt_loc, Tr * k));
    TRY_ALLOC(dalloc(&L->logits, Tr * L->E));
    TRY_ALLOC(dalloc(&L->src, L->T));
    TRY_ALLOC(dalloc(&L->dropped, L->T));
    TRY_ALLOC(dalloc(reinterpret_cast<uint8_t**>(&L->perm_ws), permute_workspace_bytes(L->T, L->E, k, L->n)));
    TRY_ALLOC(dalloc(&L->row_map_in, L->T * k));
    TRY_ALLOC(dalloc(&L->out_expert, L->T * k));
    TRY_ALLOC(dalloc(&L->out_src, L->T * k));
    TRY_ALLOC(dalloc(&L->counts, L->E));
    TRY_ALLOC(dalloc(&L->expert_off, el + 1));
    TRY_ALLOC(dalloc(&L->rows, 1));
    TRY_ALLOC(dalloc(&L->gpad_rows, el));
    TRY_ALLOC(dalloc(&L->gpad_off, el + 1));
    TRY_ALLOC(dalloc(&L->pad_tok, Mp));
    TRY_ALLOC(dalloc(&L->row_dst, Mp));
    TRY_ALLOC(dalloc(&L->row_gate, Mp));
    TRY_ALLOC(dalloc(&L->x_perm, Mp * h));
    TRY_ALLOC(dalloc(&L->fc1_out, Mp * 2 * f));
    TRY_ALLOC(dalloc(&L->fc2_in, Mp * f));
    TRY_ALLOC(dalloc(&L->dy_perm, Mp * h));
    TRY_ALLOC(dalloc(&L->dfc1, Mp * 2 * f));
    TRY_ALLOC(dalloc(&L->dgate_part, Mp * (f / 256) * 2));
    TRY_ALLOC(dalloc(&L->dlogits, Tr * L->E));
    TRY_ALLOC(dalloc(&L->ready, Mp / L->pad + 2));  // + the dispatch row-claim counter
    TRY_ALLOC(dalloc(&L->first_row, L->T));
    TRY_ALLOC(dalloc(&L->dup_src, Mp));
    TRY_ALLOC(dalloc(&L->row_done, Mp));
    TRY_ALLOC(dalloc(&L->rw_part, (L->E <= 8 ? (Tr + kRw8Chunk - 1) / kRw8Chunk : (Tr + kRwChunk - 1) / kRwChunk) *
                                      L->E * h));
    TRY_ALLOC(dalloc(&L->tab_remote, F_COUNT * L->n));
    TRY_ALLOC(dalloc(&L->tab_local, F_COUNT * L->n));
    TRY_ALLOC(dalloc(&L->err, 1));
    TRY_ALLOC(dalloc(&L->epoch_dev, 1));
    TRY_ALLOC(dalloc(&L->counters, 10));
    TRY_ALLOC(dalloc(&L->stamps, kStampSlots));
    if (L->E <= 8 && h % 256 == 0) {
        // default 1: the split (2 or 4 CTAs per 16-token block) measured slower at the
        // Mixtral shape (ncu 22 vs 13 us at 4 CTAs: 3.5 waves at 2 CTAs/SM)
        L->router_split = 1;
        if (const char* e = getenv("MOE_ROUTER_SPLIT")) {
            const int v = atoi(e);
            if (v == 1 || (v == 2 && h % 512 == 0) || (v == 4 && h % 1024 == 0)) L->router_split = v;
        }
        TRY_ALLOC(dalloc(&L->router_part, (Tr + 15) / 16 * L->router_split * 128));
        TRY_ALLOC(dalloc(&L->router_cnt, (Tr + 15) / 16));
        cudaMemset(L->router_cnt, 0, (Tr + 15) / 16 * sizeof(unsigned));
    }
    TRY_ALLOC(dalloc(&L->router_rows, 1));
    L->norm = c.ffn_norm != 0;
    if (L->norm) {
        TRY_ALLOC(dalloc(&L->x_res, Tr * h));
        TRY_ALLOC(dalloc(&L->dxn, Tr * h));
        TRY_ALLOC(dalloc(&L->gamma, h));
        TRY_ALLOC(dalloc(&L->rstd, Tr));
        TRY_ALLOC(dalloc(&L->dgamma, h));
        TRY_ALLOC(dalloc(&L->dgamma_part, ((Tr + kRwChunk - 1) / kRwChunk) * h));
    }
    TRY_ALLOC(dalloc(&L->dlogits_bf16, Tr * L->E));
    if (L->ag) {
        TRY_ALLOC(dalloc(&L->x_all, L->T * h));
        TRY_ALLOC(dalloc(&L->ag_ready, L->n * ((Tr + 63) / 64)));
        TRY_ALLOC(dalloc(&L->inv, L->T * k));
        TRY_ALLOC(dalloc(&L->rows_out, Mp * h));
    }
    cudaMemset(L->err, 0, sizeof(int));
    if (cudaHostAlloc(&L->err_host, sizeof(int), cudaHostAllocDefault) != cudaSuccess) {
        moe_layer_destroy(L);
        return set_error(MOE_ERR_CUDA, "pinned error flag allocation failed");
    }
    *L->err_host = 0;
    cudaMemset(L->epoch_dev, 0, sizeof(uint32_t));
    // Dispatch fused into fc1 / fc2-dgrad (comm warps) when there are peer rows to
    // overlap or the permuted copy is large: on one GPU with top-2 routing the
    // separate scatter kernel + plain GEMMs measured 0.06 ms per Mixtral step
    // faster (fc1 1.46 -> 1.41 ms, fc2-dgrad 0.83 -> 0.79 ms for 0.035 ms of
    // scatter kernels), while with top-8 (DeepSeek) the two 1.1 GB scatter passes
    // cost more than the comm warps (17.5 -> 17.9 ms). Gate-after-fc2 backward,
    // FP8 comm and ag_rs need the fused path. MOE_FUSED_DISPATCH=1 /
    // MOE_UNFUSED_DISPATCH=1 override.
    {
        bool fused = L->n > 1 || L->k > 2;
        if (getenv("MOE_FUSED_DISPATCH")) fused = true;
        if (getenv("MOE_UNFUSED_DISPATCH")) fused = false;
        L->fused_dispatch = fused || L->gate_after || L->fp8 || L->ag;
    }
    // on by default (DeepSeek shape, EP = 4: 9.17 -> 8.93 ms per step with the
    // dynamic tile schedule; Mixtral EP = 4 unchanged); MOE_NO_DISPATCH_DEDUP=1 off
    L->dedup = L->n > 1 && L->k > 1 && L->el > 1 && !L->ag && getenv("MOE_NO_DISPATCH_DEDUP") == nullptr;
    L->debug = getenv("MOE_DEBUG_CHECKS") != nullptr && atoi(getenv("MOE_DEBUG_CHECKS")) != 0;
    // zero the permuted buffers once so never-written rows are finite
    cudaMemset(L->x_perm, 0, Mp * h * 2);
    cudaMemset(L->dy_perm, 0, Mp * h * 2);
    cudaMemset(L->fc2_in, 0, Mp * f * 2);
    source_rank_kernel<<<64, 256>>>(L->src, (int)L->T, (int)L->Tr);
    count_launch();
    if (L->n == 1) {
        TRY_ALLOC(fill_tables(L));
        L->ipc_ready = true;
    }
    TRY_ALLOC(build_plans(L));
    for (int i = 0; i < PH_COUNT; ++i) cudaEventCreate(&L->ev[i]);
    if (cudaDeviceSynchronize() != cudaSuccess) {
        moe_layer_destroy(L);
        return set_error(MOE_ERR_CUDA, "layer init failed");
    }
#undef TRY_ALLOC
    *out = L;
    return MOE_OK;
}

void moe_layer_destroy(moe_layer* L) {
    if (!L) return;
    cudaDeviceSynchronize();
    for (int p = 0; p < (int)L->peer_arena.size(); ++p)
        if (p != L->rank && L->peer_arena[p]) cudaIpcCloseMemHandle(L->peer_arena[p]);
    void* bufs[] = {L->arena, L->w1p, L->w2, L->wr, L->ex_loc, L->gt_loc, L->logits, L->src,
                    L->dropped, L->perm_ws, L->row_map_in, L->out_expert, L->out_src, L->counts,
                    L->expert_off, L->rows, L->gpad_rows, L->gpad_off, L->pad_tok, L->row_dst,
                    L->row_gate, L->x_perm, L->fc1_out, L->fc2_in, L->dy_perm, L->dfc1,
                    L->dgate_part, L->dlogits, L->rw_part, L->ready, L->first_row, L->dup_src, L->row_done,
                    L->tab_remote, L->tab_local,
                    L->err, L->epoch_dev, L->counters, L->router_rows, L->dlogits_bf16, L->x_res, L->dxn, L->gamma, L->rstd,
                    L->dgamma, L->dgamma_part, L->x_all, L->ag_ready, L->inv, L->rows_out, L->stamps, L->router_part, L->router_cnt};
    for (void* b : bufs)
        if (b) cudaFree(b);
    for (int i = 0; i < PH_COUNT; ++i)
        if (L->ev[i]) cudaEventDestroy(L->ev[i]);
    if (L->err_host) cudaFreeHost(L->err_host);
    delete L;
}

moe_status moe_layer_set_weights(moe_layer* L, const uint16_t* d_w1, const uint16_t* d_w2,
                                 const uint16_t* d_wr, moe_stream_t stream) {
    MOE_CHECK_ARG(L && d_w1 && d_w2, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    pack_w1_kernel<<<kNumSMs * 4, 256, 0, s>>>(d_w1, L->w1p, (int)L->el, (int)L->f, (int)L->h);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    MOE_CUDA_TRY(cudaMemcpyAsync(L->w2, d_w2, L->el * L->h * L->f * 2, cudaMemcpyDeviceToDevice, s));
    if (d_wr) MOE_CUDA_TRY(cudaMemcpyAsync(L->wr, d_wr, L->E * L->h * 2, cudaMemcpyDeviceToDevice, s));
    L->weights_set = true;
    return MOE_OK;
}

uint16_t* moe_layer_input_buffer(moe_layer* L) {
    return L ? (L->norm ? L->x_res : L->mine<uint16_t>(F_X)) : nullptr;
}

uint16_t* moe_layer_dy_buffer(moe_layer* L) { return L ? L->mine<uint16_t>(F_DY) : nullptr; }

moe_status moe_layer_set_norm_weight(moe_layer* L, const float* d_gamma, moe_stream_t stream) {
    MOE_CHECK_ARG(L && d_gamma, "null argument");
    MOE_CHECK_ARG(L->norm, "layer created without ffn_norm");
    MOE_CUDA_TRY(cudaMemcpyAsync(L->gamma, d_gamma, L->h * 4, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return MOE_OK;
}

const float* moe_layer_norm_grad(moe_layer* L) { return L ? L->dgamma : nullptr; }

moe_status moe_layer_set_routing(moe_layer* L, const int32_t* d_experts, const float* d_gates,
                                 moe_stream_t stream) {
    MOE_CHECK_ARG(L && d_experts && d_gates, "null argument");
    MOE_CHECK_ARG(L->cfg.route_mode == 1, "set_routing requires route_mode = 1 (injected)");
    cudaStream_t s = (cudaStream_t)stream;
    MOE_CUDA_TRY(cudaMemcpyAsync(L->ex_loc, d_experts, L->Tr * L->k * 4, cudaMemcpyDeviceToDevice, s));
    MOE_CUDA_TRY(cudaMemcpyAsync(L->gt_loc, d_gates, L->Tr * L->k * 4, cudaMemcpyDeviceToDevice, s));
    L->routing_set = true;
    return MOE_OK;
}

// The forward in the reference's fused-pair structure (schedule.cpp:205-272):
// K1+K2 route (router, routing-metadata all-gather, capacity drop, permutation),
// K3 dispatch_fc1 (AG + local scatter fused into fc1 + SwiGLU + gate) and
// K4+K5 fc2_combine (fc2 with the gather/RS epilogue, combine).
static moe_status check_forward_args(moe_layer* L) {
    MOE_CHECK_ARG(L, "null argument");
    MOE_CHECK_ARG(L->weights_set, "weights not set");
    MOE_CHECK_ARG(L->cfg.route_mode == 0 || L->routing_set, "injected routing not set");
    MOE_CHECK_ARG(L->n == 1 || L->ipc_ready, "ep_size > 1 requires moe_layer_ipc_import");
    return pending_timeout(L);
}

static moe_status fwd_route(moe_layer* L, const uint16_t* d_x, cudaStream_t s) {
    const int64_t Tr = L->Tr, h = L->h, f = L->f, k = L->k, el = L->el;
    (void)Tr; (void)h; (void)f; (void)k; (void)el;
    uint16_t* x_sym = L->mine<uint16_t>(F_X);
    for (int i = 0; i < PH_COUNT; ++i) L->ev_used[i] = false;
    L->mark(PH_ROUTE, s);
    if (L->norm) {
        // ffn_norm: the symmetric buffer peers pull from holds the NORMALISED tokens
        if (d_x && d_x != L->x_res)
            MOE_CUDA_TRY(cudaMemcpyAsync(L->x_res, d_x, Tr * h * 2, cudaMemcpyDeviceToDevice, s));
        rmsnorm_fwd_kernel<<<kNumSMs * 4, 256, 0, s>>>(L->x_res, L->gamma, L->cfg.norm_eps, (int)Tr,
                                                       (int)h, x_sym, L->rstd);
        count_launch();
    } else if (d_x && d_x != x_sym) {
        MOE_CUDA_TRY(cudaMemcpyAsync(x_sym, d_x, Tr * h * 2, cudaMemcpyDeviceToDevice, s));
    }
    // K1 router (learned mode)
    if (L->cfg.route_mode == 0) {
        const size_t wbytes = (size_t)L->E * h * 4;  // fp32 in shared memory
        if (L->gemm_router) {
            GemmArgs a{};
            a.G = 1;
            a.group_rows = L->router_rows;
            a.N = (int)L->E;
            a.K = (int)h;
            a.b_group_stride = 0;
            a.out = L->logits;
            a.ldo = L->E;
            MOE_TRY(gemm_launch(L->p_router, a, s));
            MOE_TRY(launch_topk_from_logits(L->logits, Tr, L->E, k, L->ex_loc, L->gt_loc, s));
        } else if (L->E <= 8 && h % 256 == 0) {
            const int ns = L->router_split;
            router_logits_mma_kernel<<<(unsigned)((Tr + 15) / 16 * ns), 256, 0, s>>>(
                x_sym, L->wr, (int)Tr, (int)h, (int)L->E, L->logits, (int)k, L->ex_loc, L->gt_loc, ns,
                L->router_part, L->router_cnt);
            count_launch();
        } else if (wbytes <= 200 * 1024) {
            if (!L->router_attr) {
                MOE_CUDA_TRY(cudaFuncSetAttribute(router_logits_smem_kernel,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                L->router_attr = true;
            }
            router_logits_smem_kernel<<<kNumSMs, 256, wbytes, s>>>(x_sym, L->wr, (int)Tr, (int)h,
                                                                   (int)L->E, L->logits);
            count_launch();
            MOE_TRY(launch_topk_from_logits(L->logits, Tr, L->E, k, L->ex_loc, L->gt_loc, s));
        } else {
            MOE_TRY(launch_router_topk(x_sym, L->wr, Tr, h, L->E, k, L->logits, L->ex_loc,
                                       L->gt_loc, s));
        }
    }
    // FP8 dispatch: quantise this rank's tokens once (per-token E4M3) for the peers to pull
    if (L->fp8)
        MOE_TRY(quantize_rows(x_sym, Tr, h, true, L->mine<uint8_t>(F_X8), L->mine<float>(F_XSC), s));
    // routing metadata all-gather over NVLink
    publish_meta_kernel<<<std::min<int64_t>((Tr * k + 255) / 256, 64), 256, 0, s>>>(
        L->ex_loc, L->gt_loc, (int)(Tr * k), (int)(L->rank * Tr * k),
        L->tab<int32_t>(F_EX) + (L->comm_local ? L->rank : 0),
        L->tab<float>(F_GT) + (L->comm_local ? L->rank : 0), L->comm_local ? 1 : (int)L->n);
    count_launch();
    MOE_TRY(barrier(L, 0, s, 1));
    L->mark(PH_PERMUTE, s);
    // K2: capacity drop (replicated on every rank over the global order) + permutation
    int32_t* ex_all = L->mine<int32_t>(F_EX);
    if (L->cfg.capacity_factor > 0.0)
        MOE_TRY(launch_capacity_drop(ex_all, L->T, L->E, k, L->n, L->cfg.capacity_factor,
                                     L->dropped, s));
    else
        MOE_CUDA_TRY(cudaMemsetAsync(L->dropped, 0, L->T, s));
    MOE_TRY(launch_permute(ex_all, L->src, L->dropped, L->T, L->E, k, L->n, L->rank, L->n,
                           L->row_map_in, L->counts, L->out_expert, L->out_src, L->expert_off,
                           L->rows, L->perm_ws, L->gpad_rows, L->gpad_off, L->pad_tok, L->pad, s));
    row_info_kernel<<<(unsigned)el, 256, 0, s>>>(L->gpad_off, L->gpad_rows, L->expert_off,
                                                 L->pad_tok, L->mine<float>(F_GT), (int)k, (int)Tr,
                                                 L->row_gate, L->row_dst);
    count_launch();
    if (L->dedup) {
        MOE_CUDA_TRY(cudaMemsetAsync(L->first_row, 0x7f, L->T * 4, s));
        first_row_kernel<<<kNumSMs * 2, 256, 0, s>>>(L->pad_tok, L->gpad_off + el, (int)k, L->first_row);
        dup_src_kernel<<<kNumSMs * 2, 256, 0, s>>>(L->pad_tok, L->gpad_off + el, (int)k, L->first_row, L->dup_src);
        count_launch(2);
    }
    if (L->ag) {
        MOE_CUDA_TRY(cudaMemsetAsync(L->inv, 0xff, L->T * k * 4, s));
        inverse_rows_kernel<<<kNumSMs * 2, 256, 0, s>>>(L->pad_tok, L->gpad_off + el, L->inv);
        count_launch();
    }
    // dispatch: AG + local scatter (rows pulled from the owning rank)
    L->mark(PH_DISPATCH, s);
    if (L->fused_dispatch) {
        MOE_CUDA_TRY(cudaMemsetAsync(L->ready, 0, (L->Mp / L->pad + 2) * 4, s));
        if (L->ag) MOE_CUDA_TRY(cudaMemsetAsync(L->ag_ready, 0, L->n * ((Tr + 63) / 64) * 4, s));
        if (L->dedup) MOE_CUDA_TRY(cudaMemsetAsync(L->row_done, 0, L->Mp * 4, s));
    } else {
        dispatch_rows_kernel<<<kNumSMs * 4, 256, 0, s>>>(L->pad_tok, L->gpad_off + el, (int)k, (int)Tr,
                                                         (int)h, L->tab<const uint16_t>(F_X), L->x_perm);
        count_launch();
        MOE_CUDA_TRY(cudaGetLastError());
    }
    L->stage = 1;
    return MOE_OK;
}

static moe_status fwd_dispatch_fc1(moe_layer* L, cudaStream_t s) {
    const int64_t Tr = L->Tr, h = L->h, f = L->f, k = L->k, el = L->el;
    (void)Tr; (void)h; (void)f; (void)k; (void)el;
    // fc1 + SwiGLU (+ gate before fc2)
    L->mark(PH_FC1, s);
    {
        GemmArgs a{};
        a.G = (int)el;
        a.group_rows = L->gpad_rows;
        a.N = (int)(2 * f);
        a.K = (int)h;
        a.b_group_stride = (int)(2 * f);
        a.out = L->fc1_out;
        a.ldo = 2 * f;
        a.out2 = L->fc2_in;
        a.ldo2 = f;
        a.row_gate = L->gate_after ? nullptr : L->row_gate;
        set_dispatch(L, a, false, L->x_perm);
        GemmPlan p = L->p_fc1;
        p.dispatch = L->fused_dispatch;
        MOE_TRY(gemm_launch(p, a, s));
    }
    MOE_TRY(debug_check_dispatch(L, false, s));
    L->stage = 2;
    return MOE_OK;
}

static moe_status fwd_fc2_combine(moe_layer* L, uint16_t* d_y, cudaStream_t s) {
    const int64_t Tr = L->Tr, h = L->h, f = L->f, k = L->k, el = L->el;
    (void)Tr; (void)h; (void)f; (void)k; (void)el;
    // fc2 + gather to the source rank's combine staging (bf16 or FP8 payload)
    L->mark(PH_FC2, s);
    {
        GemmArgs a{};
        a.G = (int)el;
        a.group_rows = L->gpad_rows;
        a.N = (int)h;
        a.K = (int)f;
        a.b_group_stride = (int)h;
        a.ldo = h;
        if (L->ag) {
            // ag_rs: rows stay local; gather + reduce-scatter below
            a.out = L->rows_out;
            MOE_TRY(gemm_launch(L->p_fc2_local, a, s));
        } else {
            a.row_dst = L->row_dst;
            a.rank_base = L->fp8 ? L->tab<void>(F_STAGE8) : L->tab<void>(F_STAGE);
            a.wide_rows = L->n > 1;
            a.rank_scale_base = L->tab<void>(F_SSC);
            MOE_TRY(gemm_launch(L->p_fc2, a, s));
        }
    }
    if (L->ag) MOE_TRY(launch_gather_rs(L, s));
    MOE_TRY(barrier(L, 1, s, 0));
    // combine: fixed-order fp32 reduce over the k slots (gate after fc2 applied here)
    L->mark(PH_COMBINE, s);
    const uint8_t* drop_loc = L->dropped + L->rank * Tr;
    const float* slot_gate = L->gate_after ? L->gt_loc : nullptr;
    if (L->ag)
        combine_rs_kernel<<<kNumSMs * 4, 256, 0, s>>>(L->mine<uint16_t>(F_RSTAGE), L->ex_loc, drop_loc, (int)Tr,
                                                      (int)k, (int)el, (int)L->n, (int)h, d_y, nullptr, nullptr,
                                                      nullptr, nullptr, 0);
    else if (L->fp8)
        launch_combine<true>(s, 
            L->mine<uint8_t>(F_STAGE8), L->mine<float>(F_SSC), drop_loc, (int)Tr, (int)k, (int)h, d_y,
            slot_gate, nullptr, nullptr, nullptr, nullptr, nullptr, 0);
    else
        launch_combine<false>(s, 
            L->mine<uint16_t>(F_STAGE), nullptr, drop_loc, (int)Tr, (int)k, (int)h, d_y, slot_gate,
            nullptr, nullptr, nullptr, nullptr, nullptr, 0);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    L->mark(PH_FWD_END, s);
    MOE_TRY(mirror_error(L, s));
    L->fwd_done = true;
    L->stage = 0;
    return MOE_OK;
}

moe_status moe_layer_forward(moe_layer* L, const uint16_t* d_x, uint16_t* d_y, moe_stream_t stream) {
    MOE_CHECK_ARG(L && d_y, "null argument");
    MOE_TRY(check_forward_args(L));
    cudaStream_t s = (cudaStream_t)stream;
    MOE_TRY(fwd_route(L, d_x, s));
    MOE_TRY(fwd_dispatch_fc1(L, s));
    return fwd_fc2_combine(L, d_y, s);
}

moe_status moe_layer_route(moe_layer* L, const uint16_t* d_x, moe_stream_t stream) {
    MOE_TRY(check_forward_args(L));
    return fwd_route(L, d_x, (cudaStream_t)stream);
}

moe_status moe_dispatch_fc1(moe_layer* L, moe_stream_t stream) {
    MOE_CHECK_ARG(L, "null argument");
    MOE_CHECK_ARG(L->stage == 1, "moe_dispatch_fc1 needs moe_layer_route first");
    return fwd_dispatch_fc1(L, (cudaStream_t)stream);
}

moe_status moe_fc2_combine(moe_layer* L, uint16_t* d_y, moe_stream_t stream) {
    MOE_CHECK_ARG(L && d_y, "null argument");
    MOE_CHECK_ARG(L->stage == 2, "moe_fc2_combine needs moe_dispatch_fc1 first");
    return fwd_fc2_combine(L, d_y, (cudaStream_t)stream);
}

moe_status moe_layer_backward_ex(moe_layer* L, const uint16_t* d_dy, uint16_t* d_dx,
                                 uint16_t* d_dw1, uint16_t* d_dw2, float* d_dwr,
                                 void* dx_ready_event, moe_stream_t stream) {
    MOE_CHECK_ARG(L && d_dy && d_dx, "null argument");
    MOE_CHECK_ARG(L->fwd_done, "backward needs a preceding forward");
    MOE_TRY(pending_timeout(L));
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t Tr = L->Tr, h = L->h, f = L->f, k = L->k, el = L->el;
    uint16_t* dy_sym = L->mine<uint16_t>(F_DY);
    float* dgate_sym = L->mine<float>(F_DGATE);
    const uint8_t* drop_loc = L->dropped + L->rank * Tr;
    L->mark(PH_DISPATCH_DY, s);
    if (d_dy != dy_sym)
        MOE_CUDA_TRY(cudaMemcpyAsync(dy_sym, d_dy, Tr * h * 2, cudaMemcpyDeviceToDevice, s));
    if (L->gate_after) {
        // dgate on the source rank from the pre-gate outputs still in staging
        if (L->fp8)
            dgate_after_kernel<true><<<kNumSMs * 2, 256, 0, s>>>(dy_sym, L->mine<uint8_t>(F_STAGE8),
                                                                 L->mine<float>(F_SSC), drop_loc,
                                                                 (int)Tr, (int)k, (int)h, dgate_sym);
        else
            dgate_after_kernel<false><<<kNumSMs * 2, 256, 0, s>>>(dy_sym, L->mine<uint16_t>(F_STAGE),
                                                                  nullptr, drop_loc, (int)Tr, (int)k,
                                                                  (int)h, dgate_sym);
        count_launch();
    } else {
        // dgates of dropped (token, slot)s are never written by an expert rank
        MOE_CUDA_TRY(cudaMemsetAsync(dgate_sym, 0, Tr * k * 4, s));
    }
    if (L->fp8)
        MOE_TRY(quantize_rows(dy_sym, Tr, h, false, L->mine<uint8_t>(F_DY8), L->mine<float>(F_DYSC), s));
    MOE_TRY(barrier(L, 2, s, 1));
    // AG(dy) + scatter into permuted order (fused into the fc2 dgrad GEMM)
    if (L->fused_dispatch) {
        MOE_CUDA_TRY(cudaMemsetAsync(L->ready, 0, (L->Mp / L->pad + 2) * 4, s));
        if (L->ag) MOE_CUDA_TRY(cudaMemsetAsync(L->ag_ready, 0, L->n * ((Tr + 63) / 64) * 4, s));
        if (L->dedup && !L->gate_after) MOE_CUDA_TRY(cudaMemsetAsync(L->row_done, 0, L->Mp * 4, s));
    } else {
        dispatch_rows_kernel<<<kNumSMs * 4, 256, 0, s>>>(L->pad_tok, L->gpad_off + el, (int)k, (int)Tr,
                                                         (int)h, L->tab<const uint16_t>(F_DY), L->dy_perm);
        count_launch();
    }
    // fc2 dgrad fused with SwiGLU/gate backward and remat of fc2_in
    L->mark(PH_FC2_DGRAD, s);
    {
        GemmArgs a{};
        a.G = (int)el;
        a.group_rows = L->gpad_rows;
        a.N = (int)f;
        a.K = (int)h;
        a.b_group_stride = (int)h;
        a.out = L->dfc1;
        a.ldo = 2 * f;
        a.out2 = L->cfg.no_remat ? nullptr : L->fc2_in;   // nullptr: keep the forward's fc2_in
        a.ldo2 = f;
        a.aux = L->fc1_out;
        a.ld_aux = 2 * f;
        a.row_gate = L->gate_after ? nullptr : L->row_gate;
        a.row_part = L->gate_after ? nullptr : L->dgate_part;
        set_dispatch(L, a, true, L->dy_perm);
        GemmPlan p = L->p_fc2_dgrad;
        p.dispatch = L->fused_dispatch;
        MOE_TRY(gemm_launch(p, a, s));
    }
    MOE_TRY(debug_check_dispatch(L, true, s));
    // fc1 dgrad + gather of dx rows to the owning rank (GEMM + RS)
    L->mark(PH_FC1_DGRAD, s);
    {
        GemmArgs a{};
        a.G = (int)el;
        a.group_rows = L->gpad_rows;
        a.N = (int)h;
        a.K = (int)(2 * f);
        a.b_group_stride = (int)(2 * f);
        a.ldo = h;
        if (L->ag) {
            a.out = L->rows_out;
            MOE_TRY(gemm_launch(L->p_fc1_dgrad_local, a, s));
        } else {
            a.row_dst = L->row_dst;
            a.rank_base = L->fp8 ? L->tab<void>(F_DSTAGE8) : L->tab<void>(F_DSTAGE);
            a.wide_rows = L->n > 1;
            a.rank_scale_base = L->tab<void>(F_DSSC);
            MOE_TRY(gemm_launch(L->p_fc1_dgrad, a, s));
        }
    }
    if (L->ag) MOE_TRY(launch_gather_rs(L, s));
    L->mark(PH_DGATE, s);
    if (!L->gate_after) {
        dgate_reduce_kernel<<<kNumSMs * 4, 256, 0, s>>>(L->dgate_part, (int)(f / 256) * 2, L->row_dst,
                                                    L->gpad_off + el, L->tab<float>(F_DGATE));
        count_launch();
    }
    MOE_TRY(barrier(L, 3, s, 0));
    L->mark(PH_COMBINE_DX, s);
    const bool router = L->cfg.route_mode == 0;
    uint16_t* dx_moe = L->norm ? L->dxn : d_dx;  // gradient w.r.t. the (normalised) layer input
    if (L->ag)
        combine_rs_kernel<<<kNumSMs * 4, 256, 0, s>>>(
            L->mine<uint16_t>(F_RSTAGE), L->ex_loc, drop_loc, (int)Tr, (int)k, (int)el, (int)L->n, (int)h, dx_moe,
            router ? L->gt_loc : nullptr, router ? dgate_sym : nullptr, router ? L->wr : nullptr,
            router ? L->dlogits : nullptr, (int)L->E);
    else if (L->fp8)
        launch_combine<true>(s, 
            L->mine<uint8_t>(F_DSTAGE8), L->mine<float>(F_DSSC), drop_loc, (int)Tr, (int)k, (int)h,
            dx_moe, nullptr, router ? L->ex_loc : nullptr, router ? L->gt_loc : nullptr,
            router ? dgate_sym : nullptr, router ? L->wr : nullptr, router ? L->dlogits : nullptr,
            (int)L->E);
    else
        launch_combine<false>(s, 
            L->mine<uint16_t>(F_DSTAGE), nullptr, drop_loc, (int)Tr, (int)k, (int)h, dx_moe, nullptr,
            router ? L->ex_loc : nullptr, router ? L->gt_loc : nullptr, router ? dgate_sym : nullptr,
            router ? L->wr : nullptr, router ? L->dlogits : nullptr, (int)L->E);
    count_launch();
    if (L->norm) {
        rmsnorm_bwd_kernel<<<kNumSMs * 4, 256, 0, s>>>(L->x_res, L->gamma, L->rstd, L->dxn, (int)Tr, (int)h, d_dx);
        const int nch = (int)((Tr + kRwChunk - 1) / kRwChunk);
        rmsnorm_dgamma_partial_kernel<<<dim3((unsigned)((h + 255) / 256), nch), 256, 0, s>>>(
            L->x_res, L->rstd, L->dxn, (int)Tr, (int)h, L->dgamma_part);
        if (h % 4 == 0)
            chunk_sum4_kernel<<<(unsigned)((h / 4 + 31) / 32), 256, 0, s>>>(L->dgamma_part, nch, h, L->dgamma);
        else
            router_wgrad_reduce_kernel<<<kNumSMs, 256, 0, s>>>(L->dgamma_part, nch, 1, (int)h, L->dgamma);
        count_launch(3);
    }
    // dx is final here: callers may start its device->host copy while the
    // weight gradients below run (wgrad hidden under the dx transfer)
    if (dx_ready_event) MOE_CUDA_TRY(cudaEventRecord((cudaEvent_t)dx_ready_event, s));
    L->mark(PH_FC2_WGRAD, s);
    if (d_dw2) {
        GemmArgs a{};
        a.G = (int)el;
        a.group_rows = L->gpad_rows;
        a.N = (int)f;
        a.K = (int)h;  // output rows per expert
        a.group_k_rows = L->counts + L->first;
        a.out = d_dw2;
        a.ldo = f;
        MOE_TRY(gemm_launch(L->p_fc2_wgrad, a, s));
    }
    L->mark(PH_FC1_WGRAD, s);
    if (d_dw1) {
        GemmArgs a{};
        a.G = (int)el;
        a.group_rows = L->gpad_rows;
        a.N = (int)h;
        a.K = (int)(2 * f);
        a.group_k_rows = L->counts + L->first;
        a.out = d_dw1;
        a.ldo = h;
        a.interleave_rows = 1;
        MOE_TRY(gemm_launch(L->p_fc1_wgrad, a, s));
    }
    L->mark(PH_ROUTER_WGRAD, s);
    if (d_dwr) {
        if (router && L->gemm_router_wgrad) {
            f32_to_bf16_kernel<<<kNumSMs, 256, 0, s>>>(L->dlogits, L->dlogits_bf16, Tr * L->E);
            count_launch();
            GemmArgs a{};
            a.G = 1;
            a.group_rows = L->router_rows;
            a.N = (int)h;
            a.K = (int)L->E;  // output rows
            a.out = d_dwr;
            a.ldo = h;
            MOE_TRY(gemm_launch(L->p_router_wgrad, a, s));
        } else if (router) {
            int nch;
            if (L->E <= 8 && h % 8 == 0) {
                nch = (int)((Tr + kRw8Chunk - 1) / kRw8Chunk);
                router_wgrad_partial8_kernel<<<dim3((unsigned)((h / 8 + 127) / 128), nch), 128, 0, s>>>(
                    L->dlogits, L->mine<uint16_t>(F_X), (int)Tr, (int)h, (int)L->E, L->rw_part);
            } else {
                nch = (int)((Tr + kRwChunk - 1) / kRwChunk);
                router_wgrad_partial_kernel<32><<<dim3((unsigned)((h + 255) / 256), nch), 256, 0, s>>>(
                    L->dlogits, L->mine<uint16_t>(F_X), (int)Tr, (int)h, (int)L->E, L->rw_part);
            }
            if ((L->E * h) % 4 == 0)
                chunk_sum4_kernel<<<(unsigned)((L->E * h / 4 + 31) / 32), 256, 0, s>>>(L->rw_part, nch, L->E * h,
                                                                                    d_dwr);
            else
                router_wgrad_reduce_kernel<<<kNumSMs * 2, 256, 0, s>>>(L->rw_part, nch, (int)L->E,
                                                                       (int)h, d_dwr);
            count_launch(2);
        } else {
            MOE_CUDA_TRY(cudaMemsetAsync(d_dwr, 0, L->E * h * 4, s));
        }
    }
    MOE_CUDA_TRY(cudaGetLastError());
    MOE_TRY(mirror_error(L, s));
    L->mark(PH_END, s);
    return MOE_OK;
}

moe_status moe_layer_backward(moe_layer* L, const uint16_t* d_dy, uint16_t* d_dx, uint16_t* d_dw1,
                              uint16_t* d_dw2, float* d_dwr, moe_stream_t stream) {
    return moe_layer_backward_ex(L, d_dy, d_dx, d_dw1, d_dw2, d_dwr, nullptr, stream);
}

moe_status moe_layer_routing(moe_layer* L, moe_layer_routing_view* v) {
    MOE_CHECK_ARG(L && v, "null argument");
    v->experts = L->mine<int32_t>(F_EX);
    v->gates = L->mine<float>(F_GT);
    v->dropped = L->dropped;
    v->row_map_in = L->row_map_in;
    v->per_expert_counts = L->counts;
    v->out_expert = L->out_expert;
    v->out_source_rank = L->out_src;
    v->rows = L->rows;
    v->dgates = L->mine<float>(F_DGATE);
    v->logits = L->logits;
    return MOE_OK;
}

moe_status moe_layer_enable_timing(moe_layer* L, int enable) {
    MOE_CHECK_ARG(L, "null argument");
    L->timing = enable != 0;
    return MOE_OK;
}

moe_status moe_layer_phase_times(moe_layer* L, float* h_ms, int max_phases, int* n_phases,
                                 const char** names) {
    MOE_CHECK_ARG(L && h_ms && n_phases, "null argument");
    int last = -1;
    for (int i = 0; i < PH_COUNT; ++i)
        if (L->ev_used[i]) last = i;
    if (last < 0) return set_error(MOE_ERR_INVALID, "no timed phases recorded");
    MOE_CUDA_TRY(cudaEventSynchronize(L->ev[last]));
    int cnt = 0;
    for (int i = 0; i < PH_END && cnt < max_phases; ++i) {
        if (!L->ev_used[i] || i == PH_FWD_END) continue;
        int j = i + 1;
        while (j < PH_COUNT && !L->ev_used[j]) ++j;
        if (i == PH_COMBINE) j = PH_FWD_END;
        if (j >= PH_COUNT) break;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, L->ev[i], L->ev[j]);
        h_ms[cnt] = ms;
        if (names) names[cnt] = kPhaseNames[i];
        ++cnt;
    }
    *n_phases = cnt;
    return MOE_OK;
}

size_t moe_layer_ipc_handle_size(void) { return sizeof(cudaIpcMemHandle_t); }

moe_status moe_layer_ipc_export(moe_layer* L, void* h_blob) {
    MOE_CHECK_ARG(L && h_blob, "null argument");
    cudaIpcMemHandle_t hdl;
    MOE_CUDA_TRY(cudaIpcGetMemHandle(&hdl, L->arena));
    std::memcpy(h_blob, &hdl, sizeof(hdl));
    return MOE_OK;
}

moe_status moe_layer_ipc_import(moe_layer* L, const void* h_blobs) {
    MOE_CHECK_ARG(L && h_blobs, "null argument");
    const auto* hs = static_cast<const cudaIpcMemHandle_t*>(h_blobs);
    for (int p = 0; p < (int)L->n; ++p) {
        if (p == L->rank) continue;
        void* ptr = nullptr;
        MOE_CUDA_TRY(cudaIpcOpenMemHandle(&ptr, hs[p], cudaIpcMemLazyEnablePeerAccess));
        L->peer_arena[p] = static_cast<uint8_t*>(ptr);
    }
    MOE_TRY(fill_tables(L));
    L->ipc_ready = true;
    return MOE_OK;
}

moe_status moe_layer_set_fused_dispatch(moe_layer* L, int fused) {
    MOE_CHECK_ARG(L, "null argument");
    MOE_CHECK_ARG(fused || (!L->fp8 && !L->gate_after && !L->ag),
                  "the unfused dispatch path supports bf16 comm, gate before fc2, ep_pattern a2a only");
    L->fused_dispatch = fused != 0;
    return MOE_OK;
}

int moe_layer_get_fused_dispatch(moe_layer* L) { return L && L->fused_dispatch ? 1 : 0; }

moe_status moe_layer_set_comm_mode(moe_layer* L, int compute_only) {
    MOE_CHECK_ARG(L, "null argument");
    L->comm_local = compute_only != 0;
    return MOE_OK;
}

moe_status moe_quantize_e4m3_fast(const uint16_t* d_x, int64_t rows, int64_t cols, int32_t group,
                                  uint8_t* d_codes, float* d_scales, moe_stream_t stream) {
    MOE_CHECK_ARG(d_x && d_codes && d_scales, "null argument");
    MOE_CHECK_ARG(group == 0 || group == 128, "group must be 0 (per-token) or 128");
    MOE_CHECK_ARG(rows >= 0 && cols > 0 && cols % 128 == 0, "cols must be a positive multiple of 128");
    if (rows == 0) return MOE_OK;
    return quantize_rows(d_x, rows, cols, group == 0, d_codes, d_scales, (cudaStream_t)stream);
}

moe_status moe_layer_enable_stamps(moe_layer* L, int enable) {
    MOE_CHECK_ARG(L, "null argument");
    L->stamping = enable != 0;
    if (L->stamping) MOE_CUDA_TRY(cudaMemset(L->stamps, 0, kStampSlots * sizeof(unsigned long long)));
    return MOE_OK;
}

moe_status moe_layer_read_stamps(moe_layer* L, uint64_t* h_ns, int max_slots, int* n_phases,
                                 const char** names) {
    MOE_CHECK_ARG(L && h_ns && n_phases, "null argument");
    MOE_CUDA_TRY(cudaDeviceSynchronize());
    const int cnt = std::min(max_slots, kStampSlots);
    MOE_CUDA_TRY(cudaMemcpy(h_ns, L->stamps, cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    *n_phases = PH_COUNT;
    if (names)
        for (int i = 0; i < PH_COUNT && i < max_slots; ++i) names[i] = kPhaseNames[i];
    return MOE_OK;
}

moe_status moe_layer_status(moe_layer* L, moe_stream_t stream) {
    MOE_CHECK_ARG(L, "null argument");
    return flag_status(L->err, (cudaStream_t)stream, "moe_layer");
}

moe_status moe_layer_clear_error(moe_layer* L) {
    MOE_CHECK_ARG(L, "null argument");
    MOE_CUDA_TRY(cudaDeviceSynchronize());
    MOE_CUDA_TRY(cudaMemset(L->err, 0, sizeof(int)));
    *L->err_host = 0;
    return MOE_OK;
}

int moe_layer_error_flag(moe_layer* L) {
    int v = 0;
    if (L && L->err) cudaMemcpy(&v, L->err, sizeof(int), cudaMemcpyDeviceToHost);
    return v;
}

}  // extern "C"
