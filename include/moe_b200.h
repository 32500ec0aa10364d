/*
 * moe_b200.h — C ABI of the B200-native MegaScale-MoE layer hot path.
 *
 * One entry per operator of the reference's operator vocabulary
 * (OpKind, /root/reference/proj/core/include/moeplan/simsched.hpp:32-44;
 * node names, core/src/graph.cpp:254-311) plus the routing-map functions the
 * reference implements on the CPU (core/include/moeplan/routing.hpp:49-106)
 * and the FP8 communication quantiser (numerics.hpp:61-62), the reference's
 * numerics (round_to / quantize / emulate_reduce), the attention projections
 * of both strategies (TP: ag_attn_in/rs_attn_out, SP/Ulysses: a2a_qkv /
 * a2a_attn_out) and the compressed DP gradient sync (dp_sync_time). Each
 * declaration names the reference interface it replaces.
 *
 * Conventions
 *   - plain pointers + explicit sizes; "d_" = device pointer, "h_" = host;
 *     no C++ or torch types cross this boundary.
 *   - every call is asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) unless stated otherwise; no call synchronises the device.
 *   - index widths: token/row ids int32 on device (T*k < 2^31 at every
 *     BASELINE config); the C++ compat adapter widens to long long.
 *   - bf16 tensors are passed as uint16_t* (raw bits), row-major.
 *   - errors: a status code, never an exception (reference: domain_error ->
 *     exit 2, other -> 1, tools/src/main.cpp:595-604); moe_last_error() gives
 *     the message of the last failure on the calling thread.
 */
#ifndef MOE_B200_H
#define MOE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MOE_OK = 0,
    MOE_ERR_INTERNAL = 1,    /* reference: other std::exception -> exit 1 */
    MOE_ERR_INVALID = 2,     /* reference: std::domain_error -> exit 2 */
    MOE_ERR_CUDA = 3,
    MOE_ERR_TIMEOUT = 4,     /* cross-GPU flag wait exceeded its bound */
    MOE_ERR_UNSUPPORTED = 5
} moe_status;

typedef void* moe_stream_t; /* cudaStream_t */

const char* moe_last_error(void);
int moe_version(void);
/* Number of kernel launches this library issued on the calling process
 * since the last reset (evidence counter for bench gpu_launches). */
uint64_t moe_launch_count(void);
void moe_launch_count_reset(void);

/* ===================================================================== */
/* Routing maps (integer, bit-exact with the reference)                   */
/* ===================================================================== */

/* Group-capacity token drop.
 * Replaces: routing.cpp:113-131 (tail of simulate_routing).
 * capacity = ceil(cf * T * k / n_groups) computed in double on the host
 * exactly as routing.cpp:115-117; tokens are dropped whole, highest index
 * first, while any of their groups is over capacity.
 * d_experts[T*k] int32, d_dropped[T] uint8 out. Workspace: none. */
moe_status moe_capacity_drop(const int32_t* d_experts, int64_t T, int64_t E, int64_t k,
                             int64_t n_groups, double capacity_factor, uint8_t* d_dropped,
                             moe_stream_t stream);

/* Bytes of device workspace moe_permute needs for T tokens. */
size_t moe_permute_workspace_size(int64_t T, int64_t E, int64_t k, int64_t n_src);

/* Local-scatter row map for `my_rank`.
 * Replaces: routing::build_scatter_map (routing.hpp:72, routing.cpp:135-187).
 * Inputs: d_experts[T*k], d_source_rank[T] (values in [0, n_src)),
 *         d_dropped[T] (may be NULL = none dropped).
 * Outputs (capacity T*k rows; *h_rows/d_rows = retained local rows):
 *   d_row_map_in[rows]     = t*k + slot, ordered by (expert, source_rank, t)
 *   d_per_expert_counts[E] = retained (t,slot) per expert over ALL experts
 *   d_out_expert[rows], d_out_source_rank[rows]
 *   d_expert_offsets[E/n+1] unpadded row offsets of the local experts
 * (row_map_out is the identity and inverse_map == row_map_in in the
 * reference, routing.cpp:179-181; the adapter materialises them.)
 * Errors: MOE_ERR_INVALID unless n >= 1, 0 <= my_rank < n, E % n == 0
 * (routing.cpp:136-138). */
moe_status moe_permute(const int32_t* d_experts, const int32_t* d_source_rank,
                       const uint8_t* d_dropped, int64_t T, int64_t E, int64_t k, int64_t n,
                       int64_t my_rank, int64_t n_src, int32_t* d_row_map_in,
                       int32_t* d_per_expert_counts, int32_t* d_out_expert,
                       int32_t* d_out_source_rank, int32_t* d_expert_offsets,
                       int32_t* d_rows, void* d_workspace, moe_stream_t stream);

/* Tile slicing with per-tile dependent-source-rank sets.
 * Replaces: routing::sort_tokens_for_tiles (routing.hpp:88-89,
 * routing.cpp:189-217). Dependent ranks returned as a bitmask (ranks < 64)
 * plus the [lo, hi] window the fused dispatch waits on.
 * d_expert_offsets from moe_permute; outputs sized >= rows + E/n tiles.
 * *d_num_tiles (device) receives the tile count. */
moe_status moe_tile_layout(const int32_t* d_out_source_rank, const int32_t* d_expert_offsets,
                           int64_t num_local_experts, int64_t first_expert, int64_t tile_rows,
                           int32_t* d_tile_expert, int32_t* d_tile_begin, int32_t* d_tile_end,
                           uint64_t* d_tile_rank_mask, int32_t* d_num_tiles,
                           moe_stream_t stream);

/* Integer part of routing::balance_metrics (routing.hpp:101,
 * routing.cpp:219-262): d_per_group_load[n] (retained slots),
 * d_assigned[n] (all slots), d_dropped_tokens[1]. The host finishes the
 * double arithmetic exactly as the reference does (see the C++ adapter). */
moe_status moe_balance_counts(const int32_t* d_experts, const uint8_t* d_dropped, int64_t T,
                              int64_t E, int64_t k, int64_t n, int64_t* d_per_group_load,
                              int64_t* d_assigned, int64_t* d_dropped_tokens,
                              moe_stream_t stream);

/* ===================================================================== */
/* Router (reference node `router`, graph.cpp:268-271; cost only there)   */
/* ===================================================================== */

/* logits[T,E] = x[T,h] . wr[E,h]^T (bf16 in, fp32 accumulate); top-k by
 * logit, ties -> lower expert id, slot 0 = largest; gates = softmax over
 * the k selected logits. d_logits may be NULL. */
moe_status moe_router_topk(const uint16_t* d_x, const uint16_t* d_wr, int64_t T, int64_t h,
                           int64_t E, int64_t k, float* d_logits, int32_t* d_experts,
                           float* d_gates, moe_stream_t stream);

/* Top-k + gate softmax from given fp32 logits (bit-exact selection). */
moe_status moe_topk_from_logits(const float* d_logits, int64_t T, int64_t E, int64_t k,
                                int32_t* d_experts, float* d_gates, moe_stream_t stream);

/* ===================================================================== */
/* FP8 communication (numerics.hpp:43-62)           */
/* ===================================================================== */

/* Per-row (per_token, 1 x h) E4M3 quantisation: scale = absmax/448 (1 for
 * an all-zero row), codes = RNE(x/scale) saturating at 448.
 * Replaces: numerics::quantize(..., per_token, fp8_e4m3) for the data path.
 * x bf16 [rows, cols]; codes e4m3 bytes [rows, cols]; scales fp32 [rows]. */
moe_status moe_quantize_e4m3_rows(const uint16_t* d_x, int64_t rows, int64_t cols,
                                  uint8_t* d_codes, float* d_scales, moe_stream_t stream);
/* fp32-input variant (bit-exact against the reference's quantize on
 * fp32-representable inputs). */
moe_status moe_quantize_e4m3_rows_f32(const float* d_x, int64_t rows, int64_t cols,
                                      uint8_t* d_codes, float* d_scales, moe_stream_t stream);

/* Reference numerics, bit-exact (binary64 on the device, same operation
 * order). fmt: 0 fp32, 1 bf16, 2 fp8_e4m3 (config.hpp:41); gran: 0
 * per_tensor, 1 per_token, 2 per_channel, 3 grouped (numerics.hpp:41);
 * kind: 0 ring_bf16, 1 a2a_fp32 (numerics.hpp:64). */
/* Replaces numerics::round_to (numerics.hpp:31). */
moe_status moe_round_to(int32_t fmt, const double* d_x, int64_t n, double* d_out, moe_stream_t stream);
/* Replaces numerics::quantize (numerics.hpp:61-62): codes [rows*cols],
 * scales [moe_quantize_num_blocks(...)], workspace moe_quantize_workspace_size. */
int64_t moe_quantize_num_blocks(int64_t rows, int64_t cols, int32_t gran, int64_t group_size);
size_t moe_quantize_workspace_size(int64_t rows, int64_t cols, int32_t gran, int64_t group_size);
moe_status moe_quantize(const double* d_x, int64_t rows, int64_t cols, int32_t gran, int64_t group_size,
                        int32_t fmt, double* d_codes, double* d_scales, void* d_workspace,
                        moe_stream_t stream);
/* Replaces Quantized::dequantize (numerics.hpp:57). */
moe_status moe_dequantize(const double* d_codes, const double* d_scales, int64_t rows, int64_t cols,
                          int32_t gran, int64_t group_size, double* d_out, moe_stream_t stream);
/* Replaces numerics::emulate_reduce (numerics.hpp:77-78); vectors [ranks, dim]. */
moe_status moe_emulate_reduce(const double* d_vectors, int64_t ranks, int64_t dim, int32_t kind,
                              double* d_out, moe_stream_t stream);
/* SwiGLU a*silu(b) over [a | b] rows in binary64, optional per-row weight
 * (numerics.cpp:262-268). */
moe_status moe_swiglu_rows_f64(const double* d_x, int64_t rows, int64_t cols, const double* d_row_weight,
                               double* d_out, moe_stream_t stream);

/* ===================================================================== */
/* MoE layer (router -> dispatch -> fc1/SwiGLU -> fc2 -> combine)          */
/* ===================================================================== */

typedef struct moe_layer moe_layer; /* opaque */

typedef enum { MOE_GATE_BEFORE_FC2 = 0, MOE_GATE_AFTER_FC2 = 1 } moe_gate_order; /* numerics.hpp:86 */
typedef enum { MOE_COMM_BF16 = 0, MOE_COMM_FP8 = 1 } moe_comm_format;           /* config.hpp:41 */
typedef enum { MOE_EP_A2A = 0, MOE_EP_AG_RS = 1 } moe_ep_pattern;               /* commcost.hpp:81 (same order) */

typedef struct {
    int64_t tokens_per_rank; /* T_r (b*s/n, graph.cpp:111-113) */
    int64_t hidden;          /* h */
    int64_t ffn_hidden;      /* f (per expert) */
    int64_t num_experts;     /* E */
    int64_t top_k;           /* k */
    int64_t ep_size;         /* n (ranks) */
    int64_t rank;            /* this rank */
    double capacity_factor;  /* <= 0: no drop */
    int32_t gate_order;      /* moe_gate_order */
    int32_t comm_format;     /* moe_comm_format */
    int32_t ep_pattern;      /* moe_ep_pattern */
    int32_t route_mode;      /* 0 = learned router (K1), 1 = injected experts/gates */
    int32_t ffn_norm;        /* 1: RMSNorm (reference node ffn_norm, graph.cpp:267) fused ahead of
                                the router and the dispatch; its backward follows the dx combine */
    float norm_eps;
    int32_t no_remat;        /* 0 (reference default, RematPolicy::selective, memmodel.cpp:25-31):
                                fc2_in is recomputed from fc1_out in the fc2-dgrad epilogue;
                                1 (`--no-remat`, RematPolicy::off): the forward's fc2_in is kept
                                for the fc2 weight gradient and not rewritten */
} moe_layer_config;

moe_status moe_layer_create(const moe_layer_config* cfg, moe_layer** out);
void moe_layer_destroy(moe_layer* L);

/* Weights in the reference layout: w1 [E_local][2f][h] with rows [0,f) = a
 * and [f,2f) = b (SwiGLU = a * silu(b), numerics.cpp:262-268); w2
 * [E_local][h][f]; wr [E][h] (router, replicated). Copied into the layer's
 * HBM layout (w1 interleaved per 128-row a/b block for the fused epilogue). */
moe_status moe_layer_set_weights(moe_layer* L, const uint16_t* d_w1, const uint16_t* d_w2,
                                 const uint16_t* d_wr, moe_stream_t stream);

/* ffn_norm = 1: RMSNorm weight gamma [h] fp32 (copied). */
moe_status moe_layer_set_norm_weight(moe_layer* L, const float* d_gamma, moe_stream_t stream);
/* ffn_norm = 1: d gamma [h] fp32 of the last backward (this rank's tokens), layer-owned. */
const float* moe_layer_norm_grad(moe_layer* L);

/* Device pointer of the layer's input buffer [T_r, h] bf16 (the pre-norm
 * residual stream when ffn_norm = 1, else the symmetric buffer peers read). A
 * caller may write x there directly and pass NULL as d_x to forward. */
uint16_t* moe_layer_input_buffer(moe_layer* L);
/* Device pointer of the layer's symmetric output-gradient buffer [T_r, h] bf16
 * (peers pull dy rows from it). A caller may write dy there directly and pass
 * this pointer as d_dy to backward: no copy. */
uint16_t* moe_layer_dy_buffer(moe_layer* L);

/* Injected routing (route_mode = 1): experts [T_r, k] int32, gates [T_r, k]
 * fp32 for this rank's tokens. */
moe_status moe_layer_set_routing(moe_layer* L, const int32_t* d_experts, const float* d_gates,
                                 moe_stream_t stream);

/* Forward: y[T_r, h] = MoE(x). Retains what backward needs (fc1_out,
 * routing maps). Collective when ep_size > 1. */
moe_status moe_layer_forward(moe_layer* L, const uint16_t* d_x, uint16_t* d_y,
                             moe_stream_t stream);

/* The same forward as three operators in the reference's fused-pair
 * structure (schedule.cpp:205-272 default_fusions; FusedPair simsched.hpp:137-145),
 * issued in this order on one stream (moe_layer_forward == the three calls):
 *  - moe_layer_route   K1+K2: ffn_norm?, router + top-k + gates (graph.cpp:267-271),
 *    routing-metadata all-gather, capacity drop + build_scatter_map +
 *    tile metadata (routing.cpp:113-187);
 *  - moe_dispatch_fc1  K3: AG(+scatter)+GroupedGEMM: the token rows pulled over
 *    NVLink into permuted order inside fc1, SwiGLU (+ gate) epilogue
 *    (graph.cpp:276-295, ag_ffn_in/a2a_dispatch + scatter + fc1 + swiglu + weighted_sum);
 *  - moe_fc2_combine   K4+K5: GroupedGEMM(+gather)+RS: fc2 whose epilogue
 *    stores every row into its owner's staging over NVLink (or the ag_rs
 *    pre-reduced partials), flag barrier, fixed-order combine into d_y
 *    (graph.cpp:296-309).
 * Errors: MOE_ERR_INVALID when called out of order. */
moe_status moe_layer_route(moe_layer* L, const uint16_t* d_x, moe_stream_t stream);
moe_status moe_dispatch_fc1(moe_layer* L, moe_stream_t stream);
moe_status moe_fc2_combine(moe_layer* L, uint16_t* d_y, moe_stream_t stream);

/* Backward: dx[T_r, h] from dy[T_r, h]; weight gradients written (not
 * accumulated) into dw1 [E_local][2f][h] (reference layout), dw2
 * [E_local][h][f], dwr [E][h] (fp32, this rank's tokens' contribution).
 * Any gradient pointer may be NULL to skip it. */
moe_status moe_layer_backward(moe_layer* L, const uint16_t* d_dy, uint16_t* d_dx,
                              uint16_t* d_dw1, uint16_t* d_dw2, float* d_dwr,
                              moe_stream_t stream);

/* As moe_layer_backward; additionally records `dx_ready_event` (a
 * cudaEvent_t, may be NULL) on `stream` as soon as dx is final, before the
 * weight-gradient GEMMs, so a caller can overlap dx's transfer with them. */
moe_status moe_layer_backward_ex(moe_layer* L, const uint16_t* d_dy, uint16_t* d_dx,
                                 uint16_t* d_dw1, uint16_t* d_dw2, float* d_dwr,
                                 void* dx_ready_event, moe_stream_t stream);

/* Routing results of the last forward (device pointers owned by the layer):
 * experts/gates [T_global, k], dropped [T_global], row_map_in [rows],
 * per_expert_counts [E], out_expert/out_source_rank [rows], rows (device). */
typedef struct {
    const int32_t* experts;
    const float* gates;
    const uint8_t* dropped;
    const int32_t* row_map_in;
    const int32_t* per_expert_counts;
    const int32_t* out_expert;
    const int32_t* out_source_rank;
    const int32_t* rows;
    const float* dgates; /* after backward: [T_r, k] */
    const float* logits; /* learned-router mode: [T_r, E] */
} moe_layer_routing_view;
moe_status moe_layer_routing(moe_layer* L, moe_layer_routing_view* view);

/* Per-phase device timings of the last forward/backward (ms), measured with
 * CUDA events on the layer stream when timing is enabled. */
moe_status moe_layer_enable_timing(moe_layer* L, int enable);
moe_status moe_layer_phase_times(moe_layer* L, float* h_ms, int max_phases, int* n_phases,
                                 const char** names);

/* Measurement mode for exposed communication (reference definition
 * exposed = makespan - busy_compute, schedule.cpp:149-152): compute_only = 1
 * runs the identical kernel sequence with every peer buffer replaced by
 * this rank's own (no NVLink traffic, no cross-GPU barriers). Results are
 * not meaningful in that mode; 0 restores normal operation. */
moe_status moe_layer_set_comm_mode(moe_layer* L, int compute_only);

/* %globaltimer trace of (graph-replayed) steps: with stamps enabled, every
 * phase boundary of forward / backward records the device global timer
 * (one 1-thread kernel per boundary, captured into graphs like the rest), and
 * every cross-GPU flag barrier records its entry and release times (the wait
 * for the slowest rank = rank-imbalance idle). moe_layer_read_stamps
 * synchronises the device and copies the last step's stamps: h_ns[0..n_phases)
 * per phase (names as moe_layer_phase_times; 0 = not reached), then
 * h_ns[n_phases + 2*slot + {0, 1}] = barrier slot entry / release
 * (slots 0 metadata, 1 combine, 2 dy dispatch, 3 dx combine). */
moe_status moe_layer_enable_stamps(moe_layer* L, int enable);
moe_status moe_layer_read_stamps(moe_layer* L, uint64_t* h_ns, int max_slots, int* n_phases,
                                 const char** names);

/* 1: dispatch (AG + local scatter) fused into the fc1 / fc2-dgrad GEMMs;
 * 0: a separate memory-bound scatter kernel (the reference's unfused operator
 * structure, graph.cpp:276-286). Default: fused when ep_size > 1 or top_k > 2
 * (and always for FP8 comm, gate after fc2 and ag_rs, which need it); unfused
 * on one GPU with top-k <= 2, where there are no peer rows to overlap and the
 * separate copy is small (measured faster). */
moe_status moe_layer_set_fused_dispatch(moe_layer* L, int fused);
int moe_layer_get_fused_dispatch(moe_layer* L);

/* Non-zero if a cross-GPU flag wait of this layer timed out (synchronous). */
int moe_layer_error_flag(moe_layer* L);
/* Synchronises `stream` and returns MOE_ERR_TIMEOUT if a bounded cross-GPU
 * wait (flag barrier or fused-dispatch row arrival) of this layer gave up
 * since creation or the last moe_layer_clear_error; MOE_OK otherwise.
 * forward / backward also return MOE_ERR_TIMEOUT on entry once an earlier
 * call's timeout has reached the host (the flag is mirrored into pinned host
 * memory at the end of every multi-GPU forward / backward). */
moe_status moe_layer_status(moe_layer* L, moe_stream_t stream);
moe_status moe_layer_clear_error(moe_layer* L);

/* Generic grouped GEMM (reference OpKind::grouped_gemm): see gemm.h.
 * M-grouped: every group's row count is a multiple of 128 (also with cta_pair: a
 * group's last 128-row block then runs as an M = 128 CTA-pair tile). */
moe_status moe_grouped_gemm(const uint16_t* d_a, const uint16_t* d_b, void* d_d, int32_t groups,
                            const int32_t* d_group_rows, int64_t total_rows, int64_t M, int64_t N,
                            int64_t K, int32_t a_mn_major, int32_t b_mn_major, int32_t k_grouped,
                            int32_t out_f32, int32_t bn, int32_t cta_pair, moe_stream_t stream);

/* The layer's FP8 communication quantisers on their own (test / A-B hooks;
 * the layer calls the same kernels):
 *  - moe_quantize_e4m3_fast: the source-side quantiser of the dispatch
 *    payloads, group 0 = per-token (forward x), 128 = grouped-128 (backward
 *    dy). bf16 rows [rows, cols] -> codes [rows, cols] + fp32 scales.
 *  - moe_grouped_gemm_e4m3: the fc2 / fc1-dgrad epilogue that quantises the
 *    fp32 accumulators grouped-128 (combine payloads): M-grouped GEMM as in
 *    moe_grouped_gemm, output row r -> codes [total_rows, N] + scales
 *    [total_rows, N/128].
 * Codes equal the reference quantize (numerics.cpp:113-160: scale =
 * absmax/448 and x/scale in binary64, RNE to E4M3, saturation at 448) bit for
 * bit on the same fp32/bf16 inputs; scales are the binary64 scale rounded once
 * to fp32. */
moe_status moe_quantize_e4m3_fast(const uint16_t* d_x, int64_t rows, int64_t cols, int32_t group,
                                  uint8_t* d_codes, float* d_scales, moe_stream_t stream);
moe_status moe_grouped_gemm_e4m3(const uint16_t* d_a, const uint16_t* d_b, uint8_t* d_codes,
                                 float* d_scales, int32_t groups, const int32_t* d_group_rows,
                                 int64_t total_rows, int64_t N, int64_t K, int32_t b_mn_major,
                                 int32_t cta_pair, moe_stream_t stream);

/* ===================================================================== */
/* Multi-GPU fabric (NVLink P2P over NVSwitch; one process per GPU)       */
/* ===================================================================== */

/* Size of this rank's IPC export blob. */
size_t moe_layer_ipc_handle_size(void);
/* Export the handle of this rank's symmetric buffers (host bytes). */
moe_status moe_layer_ipc_export(moe_layer* L, void* h_blob);
/* Import all ranks' blobs (n * moe_layer_ipc_handle_size() bytes, rank
 * order) and map peer buffers. Call once after every rank exported. */
moe_status moe_layer_ipc_import(moe_layer* L, const void* h_blobs);

/* fp32 MoE layer forward on one GPU (BASELINE configs[0]): router (fp32;
 * skipped when d_experts_in/d_gates_in are given) -> capacity drop (cf <= 0:
 * none) -> permutation -> dispatch -> fc1 -> SwiGLU (-> gate) -> fc2 ->
 * gather -> combine with fp32 accuracy (relative error ~5e-6): the expert
 * GEMMs run on the tensor cores as bf16x6 (each operand split exactly into
 * three bf16 pieces; MOE_F32_FFMA=1 selects FFMA grouped GEMMs). Stateless:
 * work buffers come from the device's stream-ordered memory pool, whose
 * release threshold the first call raises so they stay cached across calls.
 * Weights in the reference layout w1 [E][2f][h] ([a|b] rows), w2 [E][h][f],
 * wr [E][h]. */
moe_status moe_ffn_forward_f32(const float* d_x, const float* d_w1, const float* d_w2,
                               const float* d_wr, int64_t T, int64_t h, int64_t f, int64_t E,
                               int64_t k, double capacity_factor, int32_t gate_order,
                               const int32_t* d_experts_in, const float* d_gates_in, float* d_y,
                               int32_t* d_experts, float* d_gates, float* d_logits,
                               uint8_t* d_dropped, moe_stream_t stream);

/* ===================================================================== */
/* Sequence-parallel attention projections (TP weights, SP activations)   */
/* reference nodes ag_attn_in + qkv_proj, out_proj + rs_attn_out,          */
/* graph.cpp:202-214; cost formulas commcost.cpp:61-64                     */
/* ===================================================================== */

typedef struct moe_attn moe_attn; /* opaque */

/* seq = full sequence length s (sharded s/tp per rank), qkv_cols_per_rank =
 * h (1 + 2/m) / tp for GQA ratio m (graph.cpp:163-165). */
moe_status moe_attn_create(int64_t seq, int64_t hidden, int64_t qkv_cols_per_rank,
                           int64_t tp_size, int64_t rank, moe_attn** out);
void moe_attn_destroy(moe_attn* A);
/* This rank's symmetric [s/tp, h] input shard buffer. */
uint16_t* moe_attn_input_buffer(moe_attn* A);
/* wqkv [qkv_cols_per_rank, h] (K-major, nn.Linear layout); wout [h, h/tp]. */
moe_status moe_attn_set_weights(moe_attn* A, const uint16_t* d_wqkv, const uint16_t* d_wout,
                                moe_stream_t stream);
/* AG-GEMM: qkv[s, qkv_cols] = AllGather_seq(x_shard) . wqkv^T, the gather
 * fused into the GEMM (in-kernel NVLink pulls gated per 256-row block).
 * d_x_shard may be NULL if the shard was written into the input buffer. */
moe_status moe_attn_ag_gemm(moe_attn* A, const uint16_t* d_x_shard, uint16_t* d_qkv,
                            moe_stream_t stream);
/* GEMM-RS: y_shard[s/tp, h] = sum over ranks of (o[s, h/tp] . wout^T), rows
 * pushed to their owner from the GEMM epilogue, fixed-order fp32 reduce. */
moe_status moe_attn_gemm_rs(moe_attn* A, const uint16_t* d_o, uint16_t* d_y_shard,
                            moe_stream_t stream);
size_t moe_attn_ipc_handle_size(void);
moe_status moe_attn_ipc_export(moe_attn* A, void* h_blob);
moe_status moe_attn_ipc_import(moe_attn* A, const void* h_blobs);
int moe_attn_error_flag(moe_attn* A);
/* Synchronises `stream`; MOE_ERR_TIMEOUT if a cross-GPU wait gave up. */
moe_status moe_attn_status(moe_attn* A, moe_stream_t stream);

/* ===================================================================== */
/* Ulysses sequence-parallel attention projections (replicated weights)     */
/* PAPER.md:150-160, 294-302; reference nodes qkv_proj -> a2a_qkv,          */
/* a2a_attn_out -> out_proj (AttnStrategy::sp, graph.cpp:189-201)          */
/* ===================================================================== */

typedef struct moe_ulysses moe_ulysses; /* opaque */

/* seq = full sequence length s (s/sp rows per rank), qkv_cols = h (1 + 2/m)
 * for GQA ratio m (graph.cpp:163-165), ordered by owning rank: rank r's head
 * group is columns [r * qkv_cols/sp, (r+1) * qkv_cols/sp). */
moe_status moe_ulysses_create(int64_t seq, int64_t hidden, int64_t qkv_cols, int64_t sp_size,
                              int64_t rank, moe_ulysses** out);
void moe_ulysses_destroy(moe_ulysses* U);
/* [s, qkv_cols/sp]: this rank's head group over the whole sequence, written by
 * moe_ulysses_qkv_a2a (symmetric; peers store into it). */
uint16_t* moe_ulysses_qkv_buffer(moe_ulysses* U);
/* [s, hidden/sp]: this rank's attention output (its heads, whole sequence),
 * read by every peer in moe_ulysses_a2a_out_proj. */
uint16_t* moe_ulysses_attn_out_buffer(moe_ulysses* U);
/* wqkv [qkv_cols, h], wout [h, h] (nn.Linear layout), replicated on every rank. */
moe_status moe_ulysses_set_weights(moe_ulysses* U, const uint16_t* d_wqkv, const uint16_t* d_wout,
                                   moe_stream_t stream);
/* GEMM + A2A: qkv = x_shard[s/sp, h] . wqkv^T with every output tile stored
 * into the rank owning its head group (fused in the GEMM epilogue). */
moe_status moe_ulysses_qkv_a2a(moe_ulysses* U, const uint16_t* d_x_shard, moe_stream_t stream);
/* A2A + GEMM: y_shard[s/sp, h] = o_seq . wout^T, where o_seq's rows are pulled
 * head group by head group from every rank's attention output inside the
 * GEMM. d_o_heads may be NULL if the output was written into the buffer. */
moe_status moe_ulysses_a2a_out_proj(moe_ulysses* U, const uint16_t* d_o_heads, uint16_t* d_y_shard,
                                    moe_stream_t stream);
size_t moe_ulysses_ipc_handle_size(void);
moe_status moe_ulysses_ipc_export(moe_ulysses* U, void* h_blob);
moe_status moe_ulysses_ipc_import(moe_ulysses* U, const void* h_blobs);
int moe_ulysses_error_flag(moe_ulysses* U);
/* Synchronises `stream`; MOE_ERR_TIMEOUT if a cross-GPU wait gave up. */
moe_status moe_ulysses_status(moe_ulysses* U, moe_stream_t stream);

/* ===================================================================== */
/* DP gradient sync with BF16 communication compression                    */
/* PAPER.md:319-334; cost commcost.cpp:182-201 (dp_sync_time, compressed); */
/* memory memmodel.cpp:112-114 (in-place operator: no transient peak)      */
/* ===================================================================== */

typedef struct moe_dp moe_dp; /* opaque */

/* count fp32 gradient elements per rank (multiple of 4096 * dp_size). */
moe_status moe_dp_create(int64_t count, int64_t dp_size, int64_t rank, moe_dp** out);
void moe_dp_destroy(moe_dp* D);
/* This rank's symmetric fp32 main-gradient buffer [count] (accumulate into it). */
float* moe_dp_grad_buffer(moe_dp* D);
/* Where moe_dp_reduce_scatter leaves this rank's reduced fp32 shard
 * [count / dp_size] (inside the gradient buffer: its upper half, or the whole
 * buffer when dp_size == 1). */
float* moe_dp_shard(moe_dp* D);
/* Compressed reduce-scatter, in place: cast the fp32 gradient to bf16 into the
 * low half of its own buffer, all-to-all the bf16 shards over NVLink, sum each
 * shard's dp_size pieces in rank order in binary64 and store fp32
 * (= numerics::emulate_reduce(a2a_fp32) then one fp32 cast, numerics.cpp:172-192).
 * The gradient buffer's contents are consumed. Collective: all ranks call. */
moe_status moe_dp_reduce_scatter(moe_dp* D, moe_stream_t stream);
/* bf16 all-gather of the updated shards: d_full[count] (bf16) receives every
 * rank's d_shard[count / dp_size] (fp32, cast to bf16 once). Collective. */
moe_status moe_dp_all_gather_bf16(moe_dp* D, const float* d_shard, uint16_t* d_full, moe_stream_t stream);
size_t moe_dp_ipc_handle_size(void);
moe_status moe_dp_ipc_export(moe_dp* D, void* h_blob);
moe_status moe_dp_ipc_import(moe_dp* D, const void* h_blobs);
int moe_dp_error_flag(moe_dp* D);
/* Synchronises `stream`; MOE_ERR_TIMEOUT if a cross-GPU wait gave up. */
moe_status moe_dp_status(moe_dp* D, moe_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* MOE_B200_H */
