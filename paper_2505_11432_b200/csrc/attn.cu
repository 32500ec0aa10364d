// attn.cu — sequence-parallel attention projections with tensor-parallel
// weights (reference nodes ag_attn_in -> qkv_proj and out_proj ->
// rs_attn_out, graph.cpp:202-214; fused-pair model schedule.cpp:205-272),
// built from the same sm_100a pieces as the MoE layer:
//
//   AG-GEMM  qkv[s, N] = AllGather_seq(x)[s, h] . Wqkv_r[N, h]^T
//            comm warps inside the tcgen05 GEMM pull the sequence shards of
//            every rank over NVLink into a local [s, h] buffer, 256-row block
//            by block, and the TMA producer waits per block (identity
//            permutation of the MoE dispatch path, k = 1).
//   GEMM-RS  y_r[s/n, h] = sum over ranks of (o[s, h/n] . Wout_r[h, h/n]^T)
//            tiles run in blocks: block c = the peer shards' tiles of output
//            column c (shards rank+1, rank+2, ...), then this rank's own tiles
//            of column c - D (decode_tile, rs_order). A peer shard's tile is
//            stored to the owner's staging slot (row, source rank) in whole
//            128-byte lines and counted on the owner's per-tile counter by the
//            CTA's signal warp; an own tile waits for its n-1 counts and its
//            epilogue sums the n partials in fixed rank order in fp32
//            (a2a_fp32 reduction semantics, numerics.cpp:172-192) straight into
//            y: no trailing barrier, no separate reduce kernel
//            (MOE_ATTN_RS_UNFUSED=1 at create: staging for every tile, flag
//            barrier, then the reduce kernel).
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <vector>

#include "gemm.h"
#include "layer_kernels.cuh"
#include "runtime.h"

using namespace moe;

struct moe_attn {
    int64_t s = 0, h = 0, nq = 0, dh = 0, n = 1, rank = 0, sr = 0;  // sr = s / n
    int cg = 2;
    uint8_t* arena = nullptr;
    size_t off_x = 0, off_stage = 0, off_flags = 0, off_rscnt = 0, arena_bytes = 0;
    std::vector<uint8_t*> peer;
    void** tab = nullptr;  // [4][n]: x shards, staging, flags, GEMM-RS tile counters
    uint16_t *x_all = nullptr, *wqkv = nullptr, *wout = nullptr;
    int32_t *ident = nullptr, *rows_s = nullptr, *rows_pad = nullptr, *row_dst = nullptr;
    uint32_t* ready = nullptr;
    uint32_t* epoch_dev = nullptr;
    uint32_t* rs_epoch = nullptr;   // GEMM-RS calls so far (the start barrier bumps it)
    bool rs_fused = true;
    int* err = nullptr;
    int* counters = nullptr;  // dynamic tile schedule, one per plan
    bool ipc_ready = false, weights = false;
    GemmPlan p_qkv, p_out;
};

namespace {

template <class T>
moe_status dalloc(T** p, size_t count) {
    MOE_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T)));
    return MOE_OK;
}

// row r of the gathered sequence is token r (k = 1); its GEMM-RS output row
// goes to the owner's staging slot (row within the owner's shard, this rank)
__global__ void attn_rows_kernel(int32_t* ident, int32_t* row_dst, int s, int sr, int n, int rank) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < s; r += gridDim.x * blockDim.x) {
        ident[r] = r;
        const int owner = r / sr;
        row_dst[r] = (owner << 27) | ((r - owner * sr) * n + rank);
    }
}

moe_status fill(moe_attn* A) {
    const int n = (int)A->n;
    std::vector<void*> t(4 * n);
    for (int p = 0; p < n; ++p) {
        t[p] = A->peer[p] + A->off_x;
        t[n + p] = A->peer[p] + A->off_stage;
        t[2 * n + p] = A->peer[p] + A->off_flags;
        t[3 * n + p] = A->peer[p] + A->off_rscnt;
    }
    MOE_CUDA_TRY(cudaMemcpy(A->tab, t.data(), sizeof(void*) * t.size(), cudaMemcpyHostToDevice));
    return MOE_OK;
}

moe_status attn_barrier(moe_attn* A, int slot, cudaStream_t s, uint32_t* epoch = nullptr) {
    if (A->n == 1) return MOE_OK;
    flag_barrier_kernel<<<1, 64, 0, s>>>(reinterpret_cast<uint32_t* const*>(A->tab + 2 * A->n), slot,
                                        (int)A->n, (int)A->rank, epoch ? epoch : A->epoch_dev, 1,
                                        flag_timeout_ns(), A->err);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

}  // namespace

extern "C" {

moe_status moe_attn_create(int64_t seq, int64_t hidden, int64_t qkv_cols_per_rank, int64_t tp_size,
                           int64_t rank, moe_attn** out) {
    MOE_CHECK_ARG(out, "null argument");
    // row destinations pack the owner as (owner << 27) into a signed int32
    // (negative = skip), so owners 0..15 round-trip
    MOE_CHECK_ARG(tp_size >= 1 && tp_size <= 16 && rank >= 0 && rank < tp_size, "bad tp_size/rank (tp_size <= 16)");
    MOE_CHECK_ARG(seq % (256 * tp_size) == 0, "seq must be a multiple of 256 * tp_size");
    MOE_CHECK_ARG(hidden % (256 * tp_size) == 0, "hidden must be a multiple of 256 * tp_size");
    MOE_CHECK_ARG(qkv_cols_per_rank % 64 == 0 && qkv_cols_per_rank >= 64, "qkv columns: multiple of 64");
    auto* A = new moe_attn();
    A->s = seq;
    A->h = hidden;
    A->nq = qkv_cols_per_rank;
    A->n = tp_size;
    A->rank = rank;
    A->sr = seq / tp_size;
    A->dh = hidden / tp_size;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off = (off + b + 255) / 256 * 256; return o; };
    A->off_x = take(A->sr * A->h * 2);
    A->off_stage = take(A->sr * A->n * A->h * 2);
    A->off_flags = take(16 * 64 * 4);
    A->off_rscnt = take((A->sr / (128 * A->cg)) * (A->h / 256) * 4);
    A->arena_bytes = off;
    A->rs_fused = getenv("MOE_ATTN_RS_UNFUSED") == nullptr;
    moe_status st;
#define TRY(expr) do { st = (expr); if (st != MOE_OK) { moe_attn_destroy(A); return st; } } while (0)
    TRY(dalloc(&A->arena, A->arena_bytes));
    cudaMemset(A->arena, 0, A->arena_bytes);
    A->peer.assign(A->n, nullptr);
    A->peer[A->rank] = A->arena;
    TRY(dalloc(&A->tab, 4 * A->n));
    TRY(dalloc(&A->x_all, A->s * A->h));
    TRY(dalloc(&A->wqkv, A->nq * A->h));
    TRY(dalloc(&A->wout, A->h * A->dh));
    TRY(dalloc(&A->ident, A->s));
    TRY(dalloc(&A->row_dst, A->s));
    TRY(dalloc(&A->rows_s, 1));
    TRY(dalloc(&A->rows_pad, 1));
    TRY(dalloc(&A->ready, A->s / 128 + 2));  // + the dispatch row-claim counter
    TRY(dalloc(&A->epoch_dev, 1));
    TRY(dalloc(&A->rs_epoch, 1));
    cudaMemset(A->rs_epoch, 0, 4);
    TRY(dalloc(&A->err, 1));
    TRY(dalloc(&A->counters, 2));
    cudaMemset(A->epoch_dev, 0, 4);
    cudaMemset(A->err, 0, 4);
    const int32_t sv = (int32_t)A->s;
    cudaMemcpy(A->rows_s, &sv, 4, cudaMemcpyHostToDevice);
    cudaMemcpy(A->rows_pad, &sv, 4, cudaMemcpyHostToDevice);
    attn_rows_kernel<<<64, 256>>>(A->ident, A->row_dst, (int)A->s, (int)A->sr, (int)A->n, (int)A->rank);
    count_launch();
    if (A->n == 1) {
        TRY(fill(A));
        A->ipc_ready = true;
    }
    // plans: AG-GEMM (A = x_all [s, h], B = wqkv [nq, h]); GEMM-RS (A = o [s, dh]
    // bound per call, B = wout [h, dh])
    A->p_qkv.cg = A->cg;
    A->p_qkv.epi = EPI_STORE_BF16;
    A->p_qkv.dispatch = true;
    {
        // tile width by wave fit: at TP = 4 (N = 2560) 256 x 256 pair tiles make
        // 320 tiles = 4.3 waves of 74 pairs (86% busy), 256 x 128 tiles 640 = 8.6
        // waves (96%) — but a 256 x 128 pair tile runs ~0.8x as fast per FLOP
        // (measured at TP = 2: AG-GEMM 0.638 vs 0.512 ms), so 128 wins only when
        // it fits the waves more than 1.25x better
        auto eff = [&](int bn) {
            const int64_t units = kNumSMs / A->cg;
            const int64_t tiles = (A->s / (128 * A->cg)) * ((A->nq + bn - 1) / bn);
            const int64_t waves = (tiles + units - 1) / units;
            return double(tiles) / double(waves * units);
        };
        A->p_qkv.bn = (A->cg == 2 && A->nq % 128 == 0 && 0.8 * eff(128) > eff(256)) ? 128 : 256;
        if (const char* e = getenv("MOE_ATTN_QKV_BN")) A->p_qkv.bn = atoi(e) == 128 && A->cg == 2 ? 128 : 256;
    }
    TRY(tmap_kmajor(&A->p_qkv.ta, A->x_all, A->s, A->h, 128));
    TRY(tmap_kmajor(&A->p_qkv.tb, A->wqkv, A->nq, A->h, A->p_qkv.bn / A->cg));
    A->p_qkv.counter = A->counters;
    A->p_out.cg = A->cg;
    A->p_out.epi = A->rs_fused ? EPI_SCATTER_RS : EPI_SCATTER;
    A->p_out.counter = A->counters + 1;
    TRY(tmap_kmajor(&A->p_out.tb, A->wout, A->h, A->dh, 256 / A->cg));
#undef TRY
    if (cudaDeviceSynchronize() != cudaSuccess) {
        moe_attn_destroy(A);
        return set_error(MOE_ERR_CUDA, "attention init failed");
    }
    *out = A;
    return MOE_OK;
}

void moe_attn_destroy(moe_attn* A) {
    if (!A) return;
    cudaDeviceSynchronize();
    for (int p = 0; p < (int)A->peer.size(); ++p)
        if (p != A->rank && A->peer[p]) cudaIpcCloseMemHandle(A->peer[p]);
    void* bufs[] = {A->arena, A->tab, A->x_all, A->wqkv, A->wout, A->ident, A->row_dst, A->rows_s,
                    A->rows_pad, A->ready, A->epoch_dev, A->rs_epoch, A->err, A->counters};
    for (void* b : bufs)
        if (b) cudaFree(b);
    delete A;
}

uint16_t* moe_attn_input_buffer(moe_attn* A) { return A ? reinterpret_cast<uint16_t*>(A->arena + A->off_x) : nullptr; }

moe_status moe_attn_set_weights(moe_attn* A, const uint16_t* d_wqkv, const uint16_t* d_wout,
                                moe_stream_t stream) {
    MOE_CHECK_ARG(A && d_wqkv && d_wout, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    MOE_CUDA_TRY(cudaMemcpyAsync(A->wqkv, d_wqkv, A->nq * A->h * 2, cudaMemcpyDeviceToDevice, s));
    MOE_CUDA_TRY(cudaMemcpyAsync(A->wout, d_wout, A->h * A->dh * 2, cudaMemcpyDeviceToDevice, s));
    A->weights = true;
    return MOE_OK;
}

moe_status moe_attn_ag_gemm(moe_attn* A, const uint16_t* d_x_shard, uint16_t* d_qkv,
                            moe_stream_t stream) {
    MOE_CHECK_ARG(A && d_qkv, "null argument");
    MOE_CHECK_ARG(A->weights && A->ipc_ready, "weights / IPC not set");
    cudaStream_t s = (cudaStream_t)stream;
    uint16_t* xs = reinterpret_cast<uint16_t*>(A->arena + A->off_x);
    if (d_x_shard && d_x_shard != xs)
        MOE_CUDA_TRY(cudaMemcpyAsync(xs, d_x_shard, A->sr * A->h * 2, cudaMemcpyDeviceToDevice, s));
    MOE_TRY(attn_barrier(A, 0, s));  // every shard is in place before peers pull it
    MOE_CUDA_TRY(cudaMemsetAsync(A->ready, 0, (A->s / 128 + 2) * 4, s));
    GemmArgs a{};
    a.G = 1;
    a.group_rows = A->rows_s;
    a.N = (int)A->nq;
    a.K = (int)A->h;
    a.out = d_qkv;
    a.ldo = A->nq;
    a.m_chunk = 4;  // first wave waits for 4 row blocks, not the whole gather
    {
        // a partial last wave of at most half the CTA pairs runs as M = 128 pair tiles
        // (TP = 4: 320 tiles = 4 waves + 24 -> the last 24 become 48 half tiles)
        const int units = kNumSMs / A->cg;
        const int tiles = (int)(A->s / (128 * A->cg)) * (int)((A->nq + A->p_qkv.bn - 1) / A->p_qkv.bn);
        const int rem = tiles % units;
        static const bool no_split = getenv("MOE_ATTN_NO_TAIL_SPLIT") != nullptr;
        if (A->cg == 2 && rem > 0 && 2 * rem <= units && !no_split) a.split_last = rem;
    }
    // start on this rank's own shard, then the next rank's (rotation): the first
    // wave needs no peer rows and every rank pulls from a different peer at a time
    a.m_rot = (int)(A->rank * A->sr / (128 * A->cg));
    a.row_rot = (int)(A->rank * A->sr);
    a.pad_row_tok = A->ident;
    a.nrows_pad = A->rows_pad;
    a.src_bufs = reinterpret_cast<const uint16_t* const*>(A->tab);
    a.a_dst = A->x_all;
    a.ready = A->ready;
    a.row_claim = reinterpret_cast<int*>(A->ready + A->s / 128 + 1);
    a.topk = 1;
    a.tokens_per_rank = (int)A->sr;
    a.err = A->err;
    return gemm_launch(A->p_qkv, a, s);
}

moe_status moe_attn_gemm_rs(moe_attn* A, const uint16_t* d_o, uint16_t* d_y_shard,
                            moe_stream_t stream) {
    MOE_CHECK_ARG(A && d_o && d_y_shard, "null argument");
    MOE_CHECK_ARG(A->weights && A->ipc_ready, "weights / IPC not set");
    cudaStream_t s = (cudaStream_t)stream;
    GemmPlan p = A->p_out;
    MOE_TRY(tmap_kmajor(&p.ta, d_o, A->s, A->dh, 128));
    GemmArgs a{};
    a.G = 1;
    a.group_rows = A->rows_s;
    a.N = (int)A->h;
    a.K = (int)A->dh;
    a.b_group_stride = 0;
    a.ldo = A->h;
    a.row_dst = A->row_dst;
    a.rank_base = reinterpret_cast<void* const*>(A->tab + A->n);
    a.wide_rows = A->n > 1;
    a.err = A->err;
    if (A->rs_fused) {
        // owners finished reading the previous call's staging; bumps the call count
        MOE_TRY(attn_barrier(A, 1, s, A->rs_epoch));   // (n = 1: nothing to wait for)
        const int tm = 128 * A->cg;
        const int n_tiles = (int)(A->h / 256);
        static const int delay_env = getenv("MOE_ATTN_RS_DELAY") ? atoi(getenv("MOE_ATTN_RS_DELAY")) : 6;
        a.rs_order = 1;
        a.rs_delay = std::max(0, std::min(delay_env, n_tiles - 1));
        a.self_rank = (int)A->rank;
        a.rs_cnt = reinterpret_cast<uint32_t* const*>(A->tab + 3 * A->n);
        a.rs_epoch = A->rs_epoch;
        a.rs_out = d_y_shard;
        a.rs_rows = (int)A->sr;
        a.rs_n = (int)A->n;
        a.rs_tile_m = tm;
        a.rs_tile_warps = 8 * A->cg;
        return gemm_launch(p, a, s);
    }
    MOE_TRY(attn_barrier(A, 1, s));  // owners finished reading the previous staging
    // m-tiles of every column start at the own shard; each column interleaves
    // all owners, so the link carries the pushes for the whole GEMM
    a.m_rot = (int)(A->rank * A->sr / (128 * A->cg));
    MOE_TRY(gemm_launch(p, a, s));
    MOE_TRY(attn_barrier(A, 2, s));
    launch_combine<false>(s,
        A->arena + A->off_stage, nullptr, nullptr, (int)A->sr, (int)A->n, (int)A->h, d_y_shard,
        nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

size_t moe_attn_ipc_handle_size(void) { return sizeof(cudaIpcMemHandle_t); }

moe_status moe_attn_ipc_export(moe_attn* A, void* h_blob) {
    MOE_CHECK_ARG(A && h_blob, "null argument");
    cudaIpcMemHandle_t hd;
    MOE_CUDA_TRY(cudaIpcGetMemHandle(&hd, A->arena));
    std::memcpy(h_blob, &hd, sizeof(hd));
    return MOE_OK;
}

moe_status moe_attn_ipc_import(moe_attn* A, const void* h_blobs) {
    MOE_CHECK_ARG(A && h_blobs, "null argument");
    const auto* hs = static_cast<const cudaIpcMemHandle_t*>(h_blobs);
    for (int p = 0; p < (int)A->n; ++p) {
        if (p == A->rank) continue;
        void* ptr = nullptr;
        MOE_CUDA_TRY(cudaIpcOpenMemHandle(&ptr, hs[p], cudaIpcMemLazyEnablePeerAccess));
        A->peer[p] = static_cast<uint8_t*>(ptr);
    }
    MOE_TRY(fill(A));
    A->ipc_ready = true;
    return MOE_OK;
}

moe_status moe_attn_status(moe_attn* A, moe_stream_t stream) {
    MOE_CHECK_ARG(A, "null argument");
    return flag_status(A->err, (cudaStream_t)stream, "moe_attn");
}

int moe_attn_error_flag(moe_attn* A) {
    int v = 0;
    if (A && A->err) cudaMemcpy(&v, A->err, sizeof(int), cudaMemcpyDeviceToHost);
    return v;
}

}  // extern "C"
