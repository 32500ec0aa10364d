// ulysses.cu — Ulysses sequence-parallel attention projections (the paper's
// chosen attention strategy; fused kernels PAPER.md:294-302;
// reference nodes qkv_proj -> a2a_qkv and a2a_attn_out -> out_proj,
// graph.cpp:189-201), on the same sm_100a GEMM as the MoE layer:
//
//   GEMM + A2A   qkv[s/n rows of this rank, all heads] = x_shard . Wqkv^T; the
//                epilogue stores every output tile straight into the rank that
//                owns its head group (columns [r*C, (r+1)*C) -> rank r, row
//                rank*s/n + i), so after one flag barrier each rank holds
//                qkv[s, C] for its heads over the whole sequence.
//   A2A + GEMM   y_shard[s/n, h] = o_seq . Wout^T where o_seq row i = the n
//                head-group pieces of sequence row rank*s/n + i, pulled from
//                every rank's [s, h/n] attention output by comm warps inside the
//                GEMM (own piece first, then the peers in rotated order) and
//                gated per 128-row block.
// Weights are replicated (SP); Wqkv's rows are ordered by owning rank (each
// rank's Q heads, then its K and V heads).
#include <cstring>
#include <vector>

#include "gemm.h"
#include "layer_kernels.cuh"
#include "runtime.h"

using namespace moe;

struct moe_ulysses {
    int64_t s = 0, h = 0, nqkv = 0, n = 1, rank = 0, sr = 0, cpo = 0, dh = 0;
    int cg = 2;
    uint8_t* arena = nullptr;
    size_t off_qkv = 0, off_o = 0, off_flags = 0, arena_bytes = 0;
    std::vector<uint8_t*> peer;
    void** tab = nullptr;  // [3][n]: qkv head buffers, attention-output buffers, flags
    uint16_t *o_seq = nullptr, *wqkv = nullptr, *wout = nullptr;
    int32_t *ident = nullptr, *rows_sr = nullptr;
    uint32_t* ready = nullptr;
    uint32_t* epoch_dev = nullptr;
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

__global__ void iota_kernel(int32_t* v, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}

moe_status fill(moe_ulysses* U) {
    const int n = (int)U->n;
    std::vector<void*> t(3 * n);
    for (int p = 0; p < n; ++p) {
        t[p] = U->peer[p] + U->off_qkv;
        t[n + p] = U->peer[p] + U->off_o;
        t[2 * n + p] = U->peer[p] + U->off_flags;
    }
    MOE_CUDA_TRY(cudaMemcpy(U->tab, t.data(), sizeof(void*) * t.size(), cudaMemcpyHostToDevice));
    return MOE_OK;
}

moe_status u_barrier(moe_ulysses* U, int slot, cudaStream_t s) {
    if (U->n == 1) return MOE_OK;
    flag_barrier_kernel<<<1, 64, 0, s>>>(reinterpret_cast<uint32_t* const*>(U->tab + 2 * U->n), slot,
                                        (int)U->n, (int)U->rank, U->epoch_dev, 1,
                                        flag_timeout_ns(), U->err);
    count_launch();
    MOE_CUDA_TRY(cudaGetLastError());
    return MOE_OK;
}

}  // namespace

extern "C" {

moe_status moe_ulysses_create(int64_t seq, int64_t hidden, int64_t qkv_cols, int64_t sp_size, int64_t rank,
                              moe_ulysses** out) {
    MOE_CHECK_ARG(out, "null argument");
    MOE_CHECK_ARG(sp_size >= 1 && sp_size <= 32 && rank >= 0 && rank < sp_size, "bad sp_size/rank");
    MOE_CHECK_ARG(seq % (128 * sp_size) == 0, "seq must be a multiple of 128 * sp_size");
    MOE_CHECK_ARG(hidden % (64 * sp_size) == 0 && hidden % 256 == 0,
                  "hidden must be a multiple of 256 and of 64 * sp_size");
    MOE_CHECK_ARG(qkv_cols % (256 * sp_size) == 0, "qkv_cols must be a multiple of 256 * sp_size");
    auto* U = new moe_ulysses();
    U->s = seq;
    U->h = hidden;
    U->nqkv = qkv_cols;
    U->n = sp_size;
    U->rank = rank;
    U->sr = seq / sp_size;
    U->cpo = qkv_cols / sp_size;
    U->dh = hidden / sp_size;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off = (off + b + 255) / 256 * 256; return o; };
    U->off_qkv = take(U->s * U->cpo * 2);
    U->off_o = take(U->s * U->dh * 2);
    U->off_flags = take(16 * 64 * 4);
    U->arena_bytes = off;
    moe_status st;
#define TRY(expr) do { st = (expr); if (st != MOE_OK) { moe_ulysses_destroy(U); return st; } } while (0)
    TRY(dalloc(&U->arena, U->arena_bytes));
    cudaMemset(U->arena, 0, U->arena_bytes);
    U->peer.assign(U->n, nullptr);
    U->peer[U->rank] = U->arena;
    TRY(dalloc(&U->tab, 3 * U->n));
    TRY(dalloc(&U->o_seq, U->sr * U->h));
    TRY(dalloc(&U->wqkv, U->nqkv * U->h));
    TRY(dalloc(&U->wout, U->h * U->h));
    TRY(dalloc(&U->ident, U->sr));
    TRY(dalloc(&U->rows_sr, 1));
    TRY(dalloc(&U->ready, U->sr / 128 + 2));  // + the dispatch row-claim counter
    TRY(dalloc(&U->epoch_dev, 1));
    TRY(dalloc(&U->err, 1));
    TRY(dalloc(&U->counters, 2));
    cudaMemset(U->epoch_dev, 0, 4);
    cudaMemset(U->err, 0, 4);
    const int32_t sv = (int32_t)U->sr;
    cudaMemcpy(U->rows_sr, &sv, 4, cudaMemcpyHostToDevice);
    iota_kernel<<<64, 256>>>(U->ident, (int)U->sr);
    count_launch();
    if (U->n == 1) {
        TRY(fill(U));
        U->ipc_ready = true;
    }
    // GEMM + A2A: A = x_shard (bound per call), B = wqkv [nqkv, h]
    U->p_qkv.cg = U->cg;
    U->p_qkv.epi = EPI_STORE_BF16;
    U->p_qkv.counter = U->counters;
    TRY(tmap_kmajor(&U->p_qkv.tb, U->wqkv, U->nqkv, U->h, 256 / U->cg));
    // A2A + GEMM: A = o_seq [sr, h] gathered in-kernel, B = wout [h, h]
    U->p_out.cg = U->cg;
    U->p_out.epi = EPI_STORE_BF16;
    U->p_out.dispatch = true;
    U->p_out.counter = U->counters + 1;
    TRY(tmap_kmajor(&U->p_out.ta, U->o_seq, U->sr, U->h, 128));
    TRY(tmap_kmajor(&U->p_out.tb, U->wout, U->h, U->h, 256 / U->cg));
#undef TRY
    if (cudaDeviceSynchronize() != cudaSuccess) {
        moe_ulysses_destroy(U);
        return set_error(MOE_ERR_CUDA, "ulysses init failed");
    }
    *out = U;
    return MOE_OK;
}

void moe_ulysses_destroy(moe_ulysses* U) {
    if (!U) return;
    cudaDeviceSynchronize();
    for (int p = 0; p < (int)U->peer.size(); ++p)
        if (p != U->rank && U->peer[p]) cudaIpcCloseMemHandle(U->peer[p]);
    void* bufs[] = {U->arena, U->tab, U->o_seq, U->wqkv, U->wout, U->ident, U->rows_sr,
                    U->ready, U->epoch_dev, U->err, U->counters};
    for (void* b : bufs)
        if (b) cudaFree(b);
    delete U;
}

uint16_t* moe_ulysses_qkv_buffer(moe_ulysses* U) {
    return U ? reinterpret_cast<uint16_t*>(U->arena + U->off_qkv) : nullptr;
}
uint16_t* moe_ulysses_attn_out_buffer(moe_ulysses* U) {
    return U ? reinterpret_cast<uint16_t*>(U->arena + U->off_o) : nullptr;
}

moe_status moe_ulysses_set_weights(moe_ulysses* U, const uint16_t* d_wqkv, const uint16_t* d_wout,
                                   moe_stream_t stream) {
    MOE_CHECK_ARG(U && d_wqkv && d_wout, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    MOE_CUDA_TRY(cudaMemcpyAsync(U->wqkv, d_wqkv, U->nqkv * U->h * 2, cudaMemcpyDeviceToDevice, s));
    MOE_CUDA_TRY(cudaMemcpyAsync(U->wout, d_wout, U->h * U->h * 2, cudaMemcpyDeviceToDevice, s));
    U->weights = true;
    return MOE_OK;
}

moe_status moe_ulysses_qkv_a2a(moe_ulysses* U, const uint16_t* d_x_shard, moe_stream_t stream) {
    MOE_CHECK_ARG(U && d_x_shard, "null argument");
    MOE_CHECK_ARG(U->weights && U->ipc_ready, "weights / IPC not set");
    cudaStream_t s = (cudaStream_t)stream;
    GemmPlan p = U->p_qkv;
    MOE_TRY(tmap_kmajor(&p.ta, d_x_shard, U->sr, U->h, 128));
    MOE_TRY(u_barrier(U, 0, s));  // every rank is done reading its previous qkv buffer
    GemmArgs a{};
    a.G = 1;
    a.group_rows = U->rows_sr;
    a.N = (int)U->nqkv;
    a.K = (int)U->h;
    a.ldo = U->cpo;
    a.col_owner_cols = (int)U->cpo;
    a.wide_rows = U->n > 1;
    a.owner_row0 = (int)(U->rank * U->sr);
    a.rank_base = reinterpret_cast<void* const*>(U->tab);
    MOE_TRY(gemm_launch(p, a, s));
    MOE_TRY(u_barrier(U, 1, s));  // every tile has landed at its owner
    return MOE_OK;
}

moe_status moe_ulysses_a2a_out_proj(moe_ulysses* U, const uint16_t* d_o_heads, uint16_t* d_y_shard,
                                    moe_stream_t stream) {
    MOE_CHECK_ARG(U && d_y_shard, "null argument");
    MOE_CHECK_ARG(U->weights && U->ipc_ready, "weights / IPC not set");
    cudaStream_t s = (cudaStream_t)stream;
    uint16_t* ob = moe_ulysses_attn_out_buffer(U);
    if (d_o_heads && d_o_heads != ob)
        MOE_CUDA_TRY(cudaMemcpyAsync(ob, d_o_heads, U->s * U->dh * 2, cudaMemcpyDeviceToDevice, s));
    MOE_TRY(u_barrier(U, 2, s));  // every rank's attention output is in place
    MOE_CUDA_TRY(cudaMemsetAsync(U->ready, 0, (U->sr / 128 + 2) * 4, s));
    GemmArgs a{};
    a.G = 1;
    a.group_rows = U->rows_sr;
    a.N = (int)U->h;
    a.K = (int)U->h;
    a.out = d_y_shard;
    a.ldo = U->h;
    a.m_chunk = 4;
    a.pad_row_tok = U->ident;
    a.nrows_pad = U->rows_sr;
    a.src_bufs = reinterpret_cast<const uint16_t* const*>(U->tab + U->n);
    a.a_dst = U->o_seq;
    a.ready = U->ready;
    a.row_claim = reinterpret_cast<int*>(U->ready + U->sr / 128 + 1);
    a.topk = 1;
    a.tokens_per_rank = (int)U->sr;
    a.err = U->err;
    a.gather_cols = (int)U->dh;
    a.n_src = (int)U->n;
    a.src_row0 = (int)(U->rank * U->sr);
    a.src_rot = (int)U->rank;
    MOE_TRY(gemm_launch(U->p_out, a, s));
    MOE_TRY(u_barrier(U, 3, s));  // peers are done pulling this rank's attention output
    return MOE_OK;
}

size_t moe_ulysses_ipc_handle_size(void) { return sizeof(cudaIpcMemHandle_t); }

moe_status moe_ulysses_ipc_export(moe_ulysses* U, void* h_blob) {
    MOE_CHECK_ARG(U && h_blob, "null argument");
    cudaIpcMemHandle_t hd;
    MOE_CUDA_TRY(cudaIpcGetMemHandle(&hd, U->arena));
    std::memcpy(h_blob, &hd, sizeof(hd));
    return MOE_OK;
}

moe_status moe_ulysses_ipc_import(moe_ulysses* U, const void* h_blobs) {
    MOE_CHECK_ARG(U && h_blobs, "null argument");
    const auto* hs = static_cast<const cudaIpcMemHandle_t*>(h_blobs);
    for (int p = 0; p < (int)U->n; ++p) {
        if (p == U->rank) continue;
        void* ptr = nullptr;
        MOE_CUDA_TRY(cudaIpcOpenMemHandle(&ptr, hs[p], cudaIpcMemLazyEnablePeerAccess));
        U->peer[p] = static_cast<uint8_t*>(ptr);
    }
    MOE_TRY(fill(U));
    U->ipc_ready = true;
    return MOE_OK;
}

moe_status moe_ulysses_status(moe_ulysses* U, moe_stream_t stream) {
    MOE_CHECK_ARG(U, "null argument");
    return flag_status(U->err, (cudaStream_t)stream, "moe_ulysses");
}

int moe_ulysses_error_flag(moe_ulysses* U) {
    int v = 0;
    if (U && U->err) cudaMemcpy(&v, U->err, sizeof(int), cudaMemcpyDeviceToHost);
    return v;
}

}  // extern "C"
