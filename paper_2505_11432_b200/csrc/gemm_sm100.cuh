// gemm_sm100.cuh — persistent, warp-specialised tcgen05 grouped GEMM for the
// expert FFN (the reference's `fc1` / `fc2` grouped_gemm nodes,
// graph.cpp:260-261,289,296, and their backward at 2x cost, graph.cpp:345).
//
//   D_g[M, N] = A_g[M, K] . B_g[N, K]^T    (bf16 in, fp32 accumulate in TMEM)
//
// Two grouping modes:
//   M-grouped (forward fc1/fc2 and both dgrads): groups are expert row
//     segments of a permuted activation matrix, each padded to a multiple of
//     the tile height; B_g is expert g's weight.
//   K-grouped (wgrads): D_g = sum over expert g's rows; the rows are the
//     contraction dimension.
// Operands are K-major or MN-major (template flags) so dgrad/wgrad read the
// forward layouts directly (no transposes in HBM).
//
// CG = 1: one CTA per tile, UMMA M=128.
// CG = 2: a CTA pair (cluster of 2, cta_group::2) per 256-row tile. Each CTA
//   loads its 128 rows of A and half of B; the leader issues M=256 UMMAs that
//   read both CTAs' shared memory, halving the per-SM operand traffic.
//
// Roles (320 threads, 1 CTA per SM, persistent over a static tile stride):
//   warp 0        : TMA producer (multi-stage smem ring, 128B swizzle; one elected lane issues)
//   warp 1        : TMEM allocator; in the leader CTA one elected lane issues tcgen05.mma
//   warps 2..9    : epilogue, two warps per TMEM lane quarter (each half of the
//                   columns); TMEM double-buffered so tile i's epilogue
//                   overlaps tile i+1's MMA.
//   warps 10..11  : fused dispatch only: comm warps filling the A rows (dispatch_warp)
//   warp 10       : EPI_SCATTER_RS only: signal warp (per-tile arrival counts at the owner)
#pragma once

#include <type_traits>

#include "common.cuh"

namespace moe {

enum EpiKind : int {
    EPI_STORE_BF16 = 0,   // D -> bf16 rows (optionally x row gate)
    EPI_STORE_F32 = 1,    // D -> fp32 rows
    EPI_SWIGLU = 2,       // fc1: store fc1_out (bf16) and fc2_in = a*silu(b)*gate
    EPI_SCATTER = 3,      // fc2 / fc1-dgrad: rows -> (rank, slot row) staging
    EPI_SWIGLU_BWD = 4,   // fc2-dgrad: SwiGLU+gate backward, remat fc2_in, dgate partials
    EPI_SCATTER_FP8 = 5,  // EPI_SCATTER with grouped-128 E4M3 payload + fp32 scales (FP8 comm)
    EPI_SCATTER_RS = 6,   // TP GEMM-RS: peer-owned tiles -> owner staging + per-tile count;
                          // own tiles (taken last) reduce the n partials into y in rank order
};

struct GemmArgs {
    int G;                      // number of groups (local experts)
    const int* group_rows;      // [G] padded rows per group (multiple of the tile height)
    const int* group_k_rows;    // K-grouped only, optional: [G] real contraction rows per group
                                // (the padding rows above them are zero, so the k loop stops at
                                // the next 64-row block instead of the padded end)
    int N;                      // output columns
    int K;                      // M-grouped: contraction length; K-grouped: output rows M
    int b_group_stride;         // B coordinate offset per group (rows or K-rows)
    // epilogue
    void* out;                  // base of D (or fc1_out for SWIGLU, dfc1 for SWIGLU_BWD)
    int64_t ldo;                // leading dimension of out (elements)
    void* out2;                 // SWIGLU: fc2_in; SWIGLU_BWD: remat fc2_in
    int64_t ldo2;
    const float* row_gate;      // [padded rows] gate per permuted row (0 for pad rows)
    const uint16_t* aux;        // SWIGLU_BWD: fc1_out (bf16 bits)
    int64_t ld_aux;
    float* row_part;            // SWIGLU_BWD: dgate partials [padded rows][2*n_tiles]
    const int* row_dst;         // SCATTER: (rank << 27) | slot_row, -1 = skip
    void* const* rank_base;     // SCATTER: per destination rank base pointer
    int gate_rows;              // 1: multiply rows by row_gate in STORE/SCATTER epilogue
    int b_box_rows;             // K-major B: rows per TMA box (0 = whole tile half)
    int m_chunk;                // M-grouped raster: m-tiles per chunk (0 = whole group, m fastest).
                                // Fused-dispatch GEMMs use small chunks so the first wave only
                                // needs the first rows to arrive.
    int m_rot;                  // M-grouped: m-tiles are taken starting at m-tile m_rot (cyclic) —
                                // TP AG-GEMM / GEMM-RS start on this rank's own sequence shard
    int row_rot;                // fused dispatch: rows are claimed starting at row row_rot (cyclic)
    int interleave_rows;        // K-grouped STORE: map packed a/b-interleaved rows back to
                                // the reference [a | b] row order (dW1)
    // fused dispatch (AG + local scatter into the A operand, DISPATCH = true)
    const int32_t* pad_row_tok;         // [padded rows] t*k+slot, -1 = pad row
    const int32_t* nrows_pad;           // device: total padded rows
    const uint16_t* const* src_bufs;    // per source rank: token rows [T_r, K]
    uint16_t* a_dst;                    // A operand base (permuted rows) written in-kernel
    uint32_t* ready;                    // [padded rows / TILE_M] rows landed per tile block
    int* row_claim;                     // rows are claimed in order from this counter (zeroed
                                        // before the launch): any resident comm warp can fill any
                                        // row, so no CTA waits on rows owned by an unscheduled CTA
    int topk, tokens_per_rank;
    int* err;                           // set to 2 on a dispatch wait timeout
    // FP8 communication
    const uint8_t* const* src_bufs8;    // per source rank: E4M3 token rows [T_r, K]
    const float* const* src_scales;     // per source rank: scales [T_r, K / src_scale_group]
    int src_scale_group;                // K (per-token) or 128 (grouped)
    const float* row_scale;             // optional extra per-permuted-row factor (gate)
    void* const* rank_scale_base;       // SCATTER_FP8: per destination rank scale base
    // Ulysses sequence parallelism (attention projections)
    int col_owner_cols;         // STORE_BF16 GEMM+A2A: output columns are owned in blocks of this
                                // many by rank n0 / col_owner_cols; rows go to that rank's buffer
                                // rank_base[owner] at row (owner_row0 + row), column n0 - base
    int owner_row0;
    int gather_cols;            // dispatch A2A+GEMM: A row = n_src pieces of gather_cols columns,
                                // piece p = row (src_row0 + pp) of source p's [*, gather_cols]
    int n_src, src_row0, src_rot;   // sources, row offset in each source, first source (rotation)
    // dispatch dedup (k > 1 experts of a token on this rank): row pp copies the
    // already-landed row dup_src[pp] (< pp) locally instead of pulling it again
    const int32_t* dup_src;     // [padded rows] earlier row of the same token, -1 = pull
    uint32_t* row_done;         // [padded rows] set once a row has landed
    // ep_pattern = ag_rs (commcost.hpp:81; graph.cpp:276-286 "ag_ffn_in" then
    // "scatter"): the comm warps first all-gather every peer's token rows into
    // the local ag_dst [n*T_r, K] (ag_rows = (n-1)*T_r claim items, peers in
    // rotation from self_rank+1), publishing ag_ready[src][64-token chunk];
    // the local scatter then reads peers' rows from ag_dst once their chunk
    // has landed and this rank's own rows from src_bufs[self_rank].
    int ag_rows, self_rank;
    uint16_t* ag_dst;
    uint32_t* ag_ready;
    // dynamic tile schedule: zeroed before the launch; the leader CTA's producer
    // takes tiles in order with an atomic and hands them to every role through a
    // shared-memory queue (nullptr = static stride schedule)
    int* tile_counter;
    // TP GEMM-RS with the reduction fused into the GEMM (EPI_SCATTER_RS; reference
    // out_proj -> rs_attn_out, graph.cpp:208-214): rows are split into owner shards
    // of rs_rows. A tile of a peer's shard is stored to that owner's staging
    // rank_base[owner] at row (local row * rs_n + self_rank), then every epilogue
    // warp adds 1 to the owner's rs_cnt[owner][tile] (release, system scope). A
    // tile of this rank's own shard waits until its counter reaches
    // *rs_epoch * (epilogue warps per tile) * (rs_n - 1), then writes
    // y = sum over ranks r (in rank order, fp32) of bf16(partial_r) to rs_out —
    // the same values and order as the unfused staging + combine.
    uint32_t* const* rs_cnt;
    const uint32_t* rs_epoch;
    uint16_t* rs_out;
    int rs_rows, rs_n;
    int rs_tile_m, rs_tile_warps;   // rows per tile, epilogue warps per tile (both CTAs)
    int wide_rows;                  // SCATTER / GEMM+A2A STORE: rows mostly go to peers -> 128-byte lines
    int split_last;                 // M-grouped, one group, CTA pairs: the last split_last tiles run as
                                    // 2 x M = 128 pair tiles each (decode_tile)
    int rs_order, rs_delay;         // 1: fused GEMM-RS tile order (decode_tile), own tiles of a
                                    // column rs_delay blocks after the peers'
};

template <int BN, int CG>
struct GemmCfg {
    static constexpr int BM = 128;            // rows per CTA
    static constexpr int TILE_M = BM * CG;    // rows per (pair) tile
    static constexpr int BK = 64;
    static constexpr int BN_CTA = BN / CG;    // B rows loaded by each CTA
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN_CTA * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int EPI_STAGE_BYTES = 8 * 2048;  // per epilogue warp: 32 x 32 bf16 transpose tile
    static constexpr int STAGES = (206 * 1024) / STAGE_BYTES > 8 ? 8 : (206 * 1024) / STAGE_BYTES;
    static constexpr int TMEM_COLS = 2 * BN;
    static constexpr int MAX_GROUPS = 256;
    static constexpr int EPI_WARPS = 8;
    static constexpr int COMM_WARPS = 2;   // only launched for the fused-dispatch variant
    static constexpr int THREADS = 64 + EPI_WARPS * 32;
    static constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + EPI_STAGE_BYTES +
                                      (2 * STAGES + 4) * 8 + 16;
};

// Tile-sequence helper shared by all roles.
struct TileInfo {
    int g, m, n, kblocks, row0;
    int half_tile;   // CG = 2, M-grouped: last tile of a group with only 128 rows -> M = 128 UMMA
};

template <int TILE_M, bool K_GROUPED>
__device__ __forceinline__ TileInfo decode_tile(int t, const int* prefix, const int* row_off,
                                                const int* kb, const GemmArgs& a, int G, int n_tiles) {
    // the last split_last pair tiles of the sequence run as two M = 128 pair tiles
    // each (rows row0 and row0 + 128): a partial last wave of full tiles becomes
    // a shorter wave of half tiles (the host only sets it when it fits one wave)
    int split_half = -1;
    if (!K_GROUPED && TILE_M == 256 && a.split_last > 0 && t >= prefix[G] - a.split_last) {
        const int u = t - (prefix[G] - a.split_last);
        t = prefix[G] - a.split_last + (u >> 1);
        split_half = u & 1;
    }
    int lo = 0, hi = G - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= t) lo = mid;
        else hi = mid - 1;
    }
    TileInfo ti;
    ti.g = lo;
    int li = t - prefix[lo];
    ti.half_tile = 0;
    if (!K_GROUPED) {
        const int rows = row_off[lo + 1] - row_off[lo];
        const int mt = (rows + TILE_M - 1) / TILE_M;
        if (a.rs_order) {
            // fused GEMM-RS order: block c = the peer shards' tiles of column c
            // (shards self+1, self+2, ...) followed by this rank's own tiles of
            // column c - D; peers reach a column D blocks before its owner
            // reduces it, and every block keeps the link busy
            const int tps = a.rs_rows / TILE_M, P = (a.rs_n - 1) * tps, D = a.rs_delay;
            int c, r;
            bool own;
            if (li < D * P) {
                c = li / P; r = li - c * P; own = false;
            } else if (li < D * P + (n_tiles - D) * (P + tps)) {
                const int l2 = li - D * P;
                c = D + l2 / (P + tps); r = l2 % (P + tps);
                own = r >= P;
                if (own) { r -= P; c -= D; }
            } else {
                const int l3 = li - D * P - (n_tiles - D) * (P + tps);
                c = n_tiles - D + l3 / tps; r = l3 % tps; own = true;
            }
            ti.n = c;
            ti.m = own ? a.self_rank * tps + r : ((a.self_rank + 1) * tps + r) % mt;
            ti.kblocks = (a.K + 63) / 64;
            ti.row0 = row_off[lo] + ti.m * TILE_M;
            return ti;
        }
        const int mc = (a.m_chunk > 0 && a.m_chunk < mt) ? a.m_chunk : mt;
        const int full = mc * n_tiles;
        const int c = li / full;
        const int r = li - c * full;
        const int cm = min(mc, mt - c * mc);
        ti.n = r / cm;
        ti.m = c * mc + (r - ti.n * cm);
        if (a.m_rot) ti.m = (ti.m + a.m_rot) % mt;
        ti.kblocks = (a.K + 63) / 64;
        ti.row0 = row_off[lo] + ti.m * TILE_M;
        ti.half_tile = TILE_M == 256 && ti.m * TILE_M + TILE_M > rows;
        if (split_half >= 0) {
            ti.row0 += split_half * 128;
            ti.half_tile = 1;
        }
    } else {
        // n fastest: a wave of tiles shares a few A panels and streams all
        // of B's (small) contraction panel from L2
        ti.n = li % n_tiles;
        ti.m = li / n_tiles;
        ti.kblocks = kb[lo];
        ti.row0 = row_off[lo];   // contraction row offset
    }
    return ti;
}

// ---- cluster / cta_group::2 helpers ----------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_cta(const void* p, uint32_t rank) {
    uint32_t out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
    return out;
}
__device__ __forceinline__ void tma_load_2d_2sm(void* smem_dst, const CUtensorMap* map,
                                                uint32_t leader_bar, int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void umma_bf16_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// ---- dynamic tile queue helpers (cluster scope) ----------------------------
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_arrive_release_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void st_shared_cluster(uint32_t cluster_addr, int v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

// TMA / expect-tx issued by one elected lane of a convergent warp
__device__ __forceinline__ void tma_load_2d_2sm_warp(void* smem_dst, const CUtensorMap* map,
                                                     uint32_t leader_bar, int32_t c0, int32_t c1) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];\n\t}" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_warp(void* smem_dst, const CUtensorMap* map,
                                                 uint64_t* bar, int32_t c0, int32_t c1) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];\n\t}" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_warp(uint64_t* bar, uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(smem_u32(bar)), "r"(bytes)
        : "memory");
}

// Warp-convergent issue: the whole warp executes the asm and elect.sync picks
// the one lane that issues, so the operands stay in (uniform) registers with
// no per-instruction broadcast loop around the MMA.
__device__ __forceinline__ void umma_bf16_2sm_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                                   uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_bf16_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit_2sm_mc_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\t.reg .pred e;\n\tmov.b16 m, 3;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}"
        ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void umma_commit_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
        ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void umma_commit_2sm_mc(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}"
        ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc_2sm(uint32_t* dst_smem) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc_2sm(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
}

// ---- coalesced row I/O through a per-warp 2 KB shared-memory tile ----------
// The accumulator gives each lane one row; global rows are far apart. These
// helpers transpose a 32-row x 32-column bf16 chunk so that every global
// access instruction covers 8 rows x 64 contiguous bytes (4 lanes per row)
// instead of 32 rows x 16 bytes. XOR swizzle on (row >> 1) & 3 keeps both
// the row-wise and the column-wise shared-memory phases conflict-free.
__device__ __forceinline__ int xs_idx(int row, int u) { return row * 4 + (u ^ ((row >> 1) & 3)); }

__device__ __forceinline__ void store_rows32(uint4* wst, const uint32_t (&pk)[16], void* row_ptr, int lane) {
#pragma unroll
    for (int u = 0; u < 4; ++u) wst[xs_idx(lane, u)] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
    __syncwarp();
    const unsigned long long my = reinterpret_cast<unsigned long long>(row_ptr);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int R = (lane >> 2) + 8 * i, c = lane & 3;
        const unsigned long long p = __shfl_sync(0xffffffffu, my, R);
        const uint4 v = wst[xs_idx(R, c)];
        if (p) reinterpret_cast<uint4*>(p)[c] = v;
    }
    __syncwarp();
}

// Same, for a warp whose 32 rows are consecutive rows `stride` bytes apart
// (every non-scatter epilogue): row addresses by arithmetic instead of shuffles.
__device__ __forceinline__ void store_rows32_s(uint4* wst, const uint32_t (&pk)[16], void* row_ptr,
                                               int64_t stride, int lane) {
#pragma unroll
    for (int u = 0; u < 4; ++u) wst[xs_idx(lane, u)] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
    __syncwarp();
    char* row0 = reinterpret_cast<char*>(row_ptr) - (int64_t)lane * stride;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int R = (lane >> 2) + 8 * i, c = lane & 3;
        reinterpret_cast<uint4*>(row0 + (int64_t)R * stride)[c] = wst[xs_idx(R, c)];
    }
    __syncwarp();
}
// 32 rows x 64 columns (bf16), each lane's row at its own address (nullptr =
// skip), in two 16-row halves of the 2 KB per-warp tile: every store
// instruction writes 4 rows x 128 contiguous bytes.
__device__ __forceinline__ void store_rows64(uint4* wst, const uint32_t (&p0)[16], const uint32_t (&p1)[16],
                                             void* row_ptr, int lane) {
    const unsigned long long my = reinterpret_cast<unsigned long long>(row_ptr);
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
        if ((lane >> 4) == hh) {
            const int r = lane & 15;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                wst[r * 8 + (u ^ (r & 7))] = make_uint4(p0[4 * u], p0[4 * u + 1], p0[4 * u + 2], p0[4 * u + 3]);
                wst[r * 8 + ((u + 4) ^ (r & 7))] = make_uint4(p1[4 * u], p1[4 * u + 1], p1[4 * u + 2], p1[4 * u + 3]);
            }
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int R = (lane >> 3) + 4 * i, c = lane & 7;
            const unsigned long long pr = __shfl_sync(0xffffffffu, my, hh * 16 + R);
            const uint4 v = wst[R * 8 + (c ^ (R & 7))];
            if (pr) reinterpret_cast<uint4*>(pr)[c] = v;
        }
        __syncwarp();
    }
}

// 32 rows x 64 columns (bf16) of consecutive rows `stride` bytes apart, through
// the same 2 KB per-warp tile in two 16-row halves: every store instruction
// writes 4 rows x 128 contiguous bytes (whole 128-byte lines: one NVLink write
// per line when the rows live on a peer).
__device__ __forceinline__ void store_rows64_s(uint4* wst, const uint32_t (&p0)[16], const uint32_t (&p1)[16],
                                               void* row_ptr, int64_t stride, int lane) {
    char* row0 = reinterpret_cast<char*>(row_ptr) - (int64_t)lane * stride;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
        if ((lane >> 4) == hh) {
            const int r = lane & 15;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                wst[r * 8 + (u ^ (r & 7))] = make_uint4(p0[4 * u], p0[4 * u + 1], p0[4 * u + 2], p0[4 * u + 3]);
                wst[r * 8 + ((u + 4) ^ (r & 7))] = make_uint4(p1[4 * u], p1[4 * u + 1], p1[4 * u + 2], p1[4 * u + 3]);
            }
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int R = (lane >> 3) + 4 * i, c = lane & 7;
            reinterpret_cast<uint4*>(row0 + (int64_t)(hh * 16 + R) * stride)[c] = wst[R * 8 + (c ^ (R & 7))];
        }
        __syncwarp();
    }
}

__device__ __forceinline__ void load_rows32_issue_s(uint4 (&v)[4], const void* row_ptr, int64_t stride, int lane) {
    const char* row0 = reinterpret_cast<const char*>(row_ptr) - (int64_t)lane * stride;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int R = (lane >> 2) + 8 * i, c = lane & 3;
        v[i] = reinterpret_cast<const uint4*>(row0 + (int64_t)R * stride)[c];
    }
}

// Same, through L2 only (.cg): rows a peer wrote over NVLink in this launch
__device__ __forceinline__ void load_rows32_issue_cg_s(uint4 (&v)[4], const void* row_ptr, int64_t stride, int lane) {
    const char* row0 = reinterpret_cast<const char*>(row_ptr) - (int64_t)lane * stride;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int R = (lane >> 2) + 8 * i, c = lane & 3;
        v[i] = __ldcg(reinterpret_cast<const uint4*>(row0 + (int64_t)R * stride) + c);
    }
}

// Issue the coalesced global loads of a 32 x 32 bf16 chunk (4 x 16 B per lane).
__device__ __forceinline__ void load_rows32_issue(uint4 (&v)[4], const void* row_ptr, int lane) {
    const unsigned long long my = reinterpret_cast<unsigned long long>(row_ptr);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int R = (lane >> 2) + 8 * i, c = lane & 3;
        const unsigned long long p = __shfl_sync(0xffffffffu, my, R);
        v[i] = reinterpret_cast<const uint4*>(p)[c];
    }
}
// ... and transpose them so this lane ends up with its own row's 16 words.
__device__ __forceinline__ void load_rows32_finish(uint4* wst, const uint4 (&v)[4], uint32_t (&pk)[16], int lane) {
#pragma unroll
    for (int i = 0; i < 4; ++i) wst[xs_idx((lane >> 2) + 8 * i, lane & 3)] = v[i];
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const uint4 x = wst[xs_idx(lane, u)];
        pk[4 * u] = x.x; pk[4 * u + 1] = x.y; pk[4 * u + 2] = x.z; pk[4 * u + 3] = x.w;
    }
    __syncwarp();
}

// ---- epilogue ---------------------------------------------------------------
// One warp handles 32 rows (its TMEM lane quarter) x `ncols` columns starting
// at column c_lo of the BN-wide accumulator.
template <int BN, int EPI, bool K_GROUPED>
__device__ __forceinline__ void epilogue_rows(const GemmArgs& args, const TileInfo& ti,
                                              int64_t orow, uint32_t tbase, int c_lo,
                                              int half, int n_tiles, uint4* wst, int tshift,
                                              uint4 (&va)[4], uint4 (&vb)[4]) {
    // accumulator column c of this warp's range lives in TMEM column c - tshift
    // (tshift = 0 except for M = 128 pair tiles)
    const int lane = threadIdx.x & 31;
    const int n0 = ti.n * BN;
    constexpr int HALF = BN / 2;
    if constexpr (EPI == EPI_STORE_BF16 || EPI == EPI_STORE_F32 || EPI == EPI_SCATTER) {
        float gscale = 1.0f;
        if (args.gate_rows) gscale = args.row_gate[orow];
        uint16_t* obf = nullptr;
        float* of32 = nullptr;
        bool valid = true;
        if (EPI == EPI_SCATTER) {
            const int dst = args.row_dst[orow];
            valid = dst >= 0;
            if (valid)
                obf = reinterpret_cast<uint16_t*>(args.rank_base[dst >> 27]) +
                      (int64_t)(dst & ((1 << 27) - 1)) * args.ldo + n0;
        } else if (EPI == EPI_STORE_BF16) {
            if (args.col_owner_cols > 0) {
                // GEMM + all-to-all: this tile's columns belong to one rank's head group
                const int owner = n0 / args.col_owner_cols;
                obf = reinterpret_cast<uint16_t*>(args.rank_base[owner]) +
                      (int64_t)(args.owner_row0 + orow) * args.ldo + (n0 - owner * args.col_owner_cols);
            } else {
                obf = reinterpret_cast<uint16_t*>(args.out) + orow * args.ldo + n0;
            }
        } else {
            of32 = reinterpret_cast<float*>(args.out) + orow * args.ldo + n0;
        }
        // peer-bound rows (scatter, GEMM + A2A with peers: args.wide_rows): 64 columns
        // per step, whole 128-byte row lines = full NVLink writes. Local stores keep
        // 32-column steps: the half-warp staging of the wide path measured 4-6% slower
        // on the short-K wgrad tiles and 1-3% on the N = 1 scatter GEMMs.
        if ((EPI == EPI_SCATTER || (EPI == EPI_STORE_BF16 && !K_GROUPED && args.col_owner_cols > 0)) &&
            args.wide_rows) {
#pragma unroll 1
            for (int c0 = c_lo; c0 < c_lo + HALF; c0 += 64) {
                if (n0 + c0 >= args.N) break;   // warp-uniform
                uint32_t r[32], p0[16], p1[16];
                tmem_ld32(tbase + (c0 - tshift), r);
                tmem_ld_wait();
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    p0[q] = pack_bf16x2(__uint_as_float(r[2 * q]) * gscale, __uint_as_float(r[2 * q + 1]) * gscale);
                if (n0 + c0 + 64 > args.N) {   // a last 32-column chunk
                    if (EPI == EPI_SCATTER) store_rows32(wst, p0, valid ? (void*)(obf + c0) : nullptr, lane);
                    else store_rows32_s(wst, p0, obf + c0, args.ldo * 2, lane);
                    break;
                }
                tmem_ld32(tbase + (c0 + 32 - tshift), r);
                tmem_ld_wait();
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    p1[q] = pack_bf16x2(__uint_as_float(r[2 * q]) * gscale, __uint_as_float(r[2 * q + 1]) * gscale);
                if (EPI == EPI_SCATTER) store_rows64(wst, p0, p1, valid ? (void*)(obf + c0) : nullptr, lane);
                else store_rows64_s(wst, p0, p1, obf + c0, args.ldo * 2, lane);
            }
            return;
        }
#pragma unroll 1
        for (int c0 = c_lo; c0 < c_lo + HALF; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tbase + (c0 - tshift), r);
            tmem_ld_wait();
            if (n0 + c0 >= args.N) continue;   // warp-uniform
            if constexpr (EPI != EPI_STORE_F32) {
                uint32_t pk[16];
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    pk[q] = pack_bf16x2(__uint_as_float(r[2 * q]) * gscale, __uint_as_float(r[2 * q + 1]) * gscale);
                if (EPI == EPI_SCATTER) store_rows32(wst, pk, valid ? (void*)(obf + c0) : nullptr, lane);
                else store_rows32_s(wst, pk, obf + c0, args.ldo * 2, lane);
            } else {
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                    float4 v = make_float4(__uint_as_float(r[i]) * gscale, __uint_as_float(r[i + 1]) * gscale,
                                           __uint_as_float(r[i + 2]) * gscale, __uint_as_float(r[i + 3]) * gscale);
                    *reinterpret_cast<float4*>(of32 + c0 + i) = v;
                }
            }
        }
    } else if constexpr (EPI == EPI_SCATTER_FP8) {
        // one warp-half = one 128-column group: absmax pass over TMEM, then
        // quantise pass; codes + one fp32 scale per (row, group) go to the
        // owning rank's staging (grouped-128 E4M3, numerics.cpp:88-160)
        static_assert(HALF == 128, "FP8 scatter needs 128-column groups");
        const int dst = args.row_dst[orow];
        float amax = 0.0f;
#pragma unroll 1
        for (int c0 = c_lo; c0 < c_lo + HALF; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tbase + (c0 - tshift), r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) amax = fmaxf(amax, fabsf(__uint_as_float(r[i])));
        }
        // binary64 scale and reference-exact codes (numerics.cpp:149-156; common.cuh)
        const E4m3Block blk = e4m3_block(amax);
        uint8_t* codes = nullptr;
        if (dst >= 0) {
            const int64_t drow = dst & ((1 << 27) - 1);
            codes = reinterpret_cast<uint8_t*>(args.rank_base[dst >> 27]) + drow * args.ldo + n0;
            reinterpret_cast<float*>(args.rank_scale_base[dst >> 27])[drow * (args.ldo / 128) + (n0 + c_lo) / 128] =
                (float)blk.scale;
        }
        // the group's 128 codes of every row are stored as one 128-byte line
        // (8 lanes per row through the per-warp tile: whole NVLink writes)
        uint32_t p0[16], p1[16];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
            uint32_t r[32];
            tmem_ld32(tbase + (c_lo + 32 * ch - tshift), r);
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint16_t lo = e4m3x2_code(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), blk);
                const uint16_t hi = e4m3x2_code(__uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]), blk);
                const uint32_t w = (uint32_t)lo | ((uint32_t)hi << 16);
                if (ch < 2) p0[8 * ch + q] = w;
                else p1[8 * (ch - 2) + q] = w;
            }
        }
        store_rows64(wst, p0, p1, dst >= 0 ? (void*)(codes + c_lo) : nullptr, lane);
    } else if constexpr (EPI == EPI_SCATTER_RS) {
        const int nr = args.rs_n, self = args.self_rank;
        const int owner = ti.row0 / args.rs_rows;
        const int64_t lrow = orow - (int64_t)owner * args.rs_rows;
        const int64_t sstride = (int64_t)nr * args.ldo * 2;   // bytes between a warp's staging rows
        if (owner != self) {
            uint16_t* obf = reinterpret_cast<uint16_t*>(args.rank_base[owner]) + (lrow * nr + self) * args.ldo + n0;
#pragma unroll 1
            for (int c0 = c_lo; c0 < c_lo + HALF; c0 += 64) {
                uint32_t r[32], p0[16], p1[16];
                tmem_ld32(tbase + (c0 - tshift), r);
                tmem_ld_wait();
#pragma unroll
                for (int q = 0; q < 16; ++q) p0[q] = pack_bf16x2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
                tmem_ld32(tbase + (c0 + 32 - tshift), r);
                tmem_ld_wait();
#pragma unroll
                for (int q = 0; q < 16; ++q) p1[q] = pack_bf16x2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
                store_rows64_s(wst, p0, p1, obf + c0, sstride, lane);
            }
        } else {
            if (lane == 0 && nr > 1) {
                const int idx = (ti.m - owner * (args.rs_rows / args.rs_tile_m)) * n_tiles + ti.n;
                const uint32_t target = *args.rs_epoch * (uint32_t)args.rs_tile_warps * (uint32_t)(nr - 1);
                const uint32_t* cnt = args.rs_cnt[self] + idx;
                const uint64_t t0 = globaltimer();
                while ((int32_t)(ld_acquire_sys(cnt) - target) < 0) {
                    if (globaltimer() - t0 > 4000000000ull) {
                        atomicExch(args.err, 4);
                        break;
                    }
                }
            }
            __syncwarp();
            const uint16_t* stage = reinterpret_cast<const uint16_t*>(args.rank_base[self]) + lrow * nr * args.ldo + n0;
            uint16_t* y = args.rs_out + lrow * args.ldo + n0;
#pragma unroll 1
            for (int c0 = c_lo; c0 < c_lo + HALF; c0 += 32) {
                uint32_t own[16];
                {
                    uint32_t r[32];
                    tmem_ld32(tbase + (c0 - tshift), r);
                    tmem_ld_wait();
#pragma unroll
                    for (int q = 0; q < 16; ++q) own[q] = pack_bf16x2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
                }
                float acc[32];
#pragma unroll
                for (int q = 0; q < 32; ++q) acc[q] = 0.0f;
                // fixed rank order, fp32 sum of bf16 partials (combine_reduce_kernel)
#pragma unroll 1
                for (int s0 = 0; s0 < nr; s0 += 4) {
                    uint4 v[4][4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int src = s0 + j;
                        if (src < nr && src != self) load_rows32_issue_cg_s(v[j], stage + src * args.ldo + c0, sstride, lane);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int src = s0 + j;
                        if (src >= nr) break;
                        uint32_t w[16];
                        if (src == self) {
#pragma unroll
                            for (int q = 0; q < 16; ++q) w[q] = own[q];
                        } else {
                            load_rows32_finish(wst, v[j], w, lane);
                        }
#pragma unroll
                        for (int q = 0; q < 16; ++q) {
                            const float2 f = unpack_bf16x2(w[q]);
                            acc[2 * q] += f.x;
                            acc[2 * q + 1] += f.y;
                        }
                    }
                }
                uint32_t pk[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) pk[q] = pack_bf16x2(acc[2 * q], acc[2 * q + 1]);
                store_rows32_s(wst, pk, y + c0, args.ldo * 2, lane);
            }
        }
    } else if constexpr (EPI == EPI_SWIGLU) {
        // W1 rows are packed per 128-row block as [a 64 | b 64] (pack_w1_kernel),
        // so this warp's accumulator columns [c_lo, c_lo + 128) hold the a/b
        // pairs of f-features ti.n * 128 + half * 64 + [0, 64). fc1_out is kept
        // in this packed column order.
        static_assert(BN == 256, "SwiGLU epilogue pairs a/b inside 128-column halves");
        const float g = args.row_gate ? args.row_gate[orow] : 1.0f;
        uint16_t* o1 = reinterpret_cast<uint16_t*>(args.out) + orow * args.ldo + n0 + c_lo;
        uint16_t* o2 = reinterpret_cast<uint16_t*>(args.out2) + orow * args.ldo2 + ti.n * HALF + half * (HALF / 2);
        const uint32_t tb = tbase + (c_lo - tshift);
#pragma unroll 1
        for (int c0 = 0; c0 < HALF / 2; c0 += 32) {
            uint32_t ra[32], rb[32];
            tmem_ld32(tb + c0, ra);
            tmem_ld32(tb + HALF / 2 + c0, rb);
            tmem_ld_wait();
            uint32_t pa[16], pb[16], ph[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                pa[q] = pack_bf16x2(__uint_as_float(ra[2 * q]), __uint_as_float(ra[2 * q + 1]));
                pb[q] = pack_bf16x2(__uint_as_float(rb[2 * q]), __uint_as_float(rb[2 * q + 1]));
                // SwiGLU on the bf16-rounded fc1_out so backward remat is exact
                const float2 a2 = unpack_bf16x2(pa[q]);
                const float2 b2 = unpack_bf16x2(pb[q]);
                ph[q] = pack_bf16x2(a2.x * silu_f(b2.x) * g, a2.y * silu_f(b2.y) * g);
            }
            store_rows32_s(wst, pa, o1 + c0, args.ldo * 2, lane);
            store_rows32_s(wst, pb, o1 + HALF / 2 + c0, args.ldo * 2, lane);
            store_rows32_s(wst, ph, o2 + c0, args.ldo2 * 2, lane);
        }
    } else if constexpr (EPI == EPI_SWIGLU_BWD) {
        // D = d fc2_in for f-columns [n0 + c_lo, +BN/2). fc1_out / dfc1 use the
        // packed [a-block(64) | b-block(64)] column order of W1.
        const float g = args.row_gate ? args.row_gate[orow] : 1.0f;
        const uint16_t* f1 = args.aux + orow * args.ld_aux;
        uint16_t* d1 = reinterpret_cast<uint16_t*>(args.out) + orow * args.ldo;
        uint16_t* rf = args.out2 ? reinterpret_cast<uint16_t*>(args.out2) + orow * args.ldo2 : nullptr;
        float dg = 0.0f;
        // va / vb: the first chunk's fc1_out rows, issued by the caller before it
        // waited for the accumulator; chunk c+1's loads fly during chunk c's stores
#pragma unroll 1
        for (int c0 = c_lo; c0 < c_lo + HALF; c0 += 32) {
            const int j = n0 + c0;           // f column
            const int ia = (j >> 6) * 128 + (j & 63);
            uint32_t aw[16], bw[16];
            load_rows32_finish(wst, va, aw, lane);
            load_rows32_finish(wst, vb, bw, lane);
            uint32_t r[32];
            tmem_ld32(tbase + (c0 - tshift), r);
            tmem_ld_wait();
            uint32_t da[16], db[16], hf[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const float2 a2 = unpack_bf16x2(aw[q]);
                const float2 b2 = unpack_bf16x2(bw[q]);
                const float d0 = __uint_as_float(r[2 * q]), d1v = __uint_as_float(r[2 * q + 1]);
                const float s0 = sigmoid_f(b2.x), s1 = sigmoid_f(b2.y);
                const float si0 = b2.x * s0, si1 = b2.y * s1;
                dg += d0 * a2.x * si0 + d1v * a2.y * si1;
                da[q] = pack_bf16x2(d0 * g * si0, d1v * g * si1);
                db[q] = pack_bf16x2(d0 * g * a2.x * s0 * (1.0f + b2.x * (1.0f - s0)),
                                    d1v * g * a2.y * s1 * (1.0f + b2.y * (1.0f - s1)));
                hf[q] = pack_bf16x2(a2.x * si0 * g, a2.y * si1 * g);
            }
            // the next chunk's fc1_out loads fly while this chunk's rows are stored
            if (c0 + 32 < c_lo + HALF) {
                const int jn = j + 32;
                const int ian = (jn >> 6) * 128 + (jn & 63);
                load_rows32_issue(va, f1 + ian, lane);
                load_rows32_issue(vb, f1 + ian + 64, lane);
            }
            store_rows32(wst, da, d1 + ia, lane);
            store_rows32(wst, db, d1 + ia + 64, lane);
            if (rf) store_rows32(wst, hf, rf + j, lane);   // remat (RematPolicy::selective)
        }
        if (args.row_part) args.row_part[orow * (2 * n_tiles) + ti.n * 2 + half] = dg;
    }
}

// Fused dispatch: COMM_WARPS extra warps per CTA pull the permuted A rows
// (from the owning rank's buffer; peers over NVLink) in padded-row order,
// and publish per-tile-block arrival counts; the TMA producer waits for its
// tile block's count before loading (tile-level AG -> GEMM overlap, the
// reference's AG+scatter+GroupedGEMM fused pair, schedule.cpp:225-242).
template <int TILE_M>
__device__ __forceinline__ void dispatch_warp(const GemmArgs& a, int K, int lane) {
    const int total = *a.nrows_pad;
    const int nvec = K / 8;
    // Rows are claimed CLAIM at a time in increasing order by whichever comm
    // warp asks next. Every claimed row belongs to a running warp and the only
    // wait inside a row (dedup: row_done[ds], ds < pp) points at an earlier
    // claim, so the rows every tile waits for always arrive, whatever subset of
    // the grid is resident (another stream may hold SMs).
    constexpr int CLAIM = 4;
    const int nag = a.ag_rows;   // all-gather items come first in the claim order
    const int Tr = a.tokens_per_rank;
    for (;;) {
    int base = 0;
    if (lane == 0) base = atomicAdd(a.row_claim, CLAIM);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= nag + total) break;
    if (base < nag) {
        // ---- AG: peer rows -> local ag_dst (NVLink pulls), rank rotation ----
        const int q_end = min(base + CLAIM, nag);
        for (int q = base; q < q_end; ++q) {
            const int pi = q / Tr, tl = q - pi * Tr;
            const int src = (a.self_rank + 1 + pi) % a.n_src;
            const uint4* sp = reinterpret_cast<const uint4*>(a.src_bufs[src] + (int64_t)tl * K);
            uint4* dp = reinterpret_cast<uint4*>(a.ag_dst + ((int64_t)src * Tr + tl) * K);
            constexpr int U = 8;   // 4 KB per warp in flight (16 would spill: comm warps share the 168-reg cap)
            for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
                uint4 r[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (v0 + 32 * u < nvec) r[u] = __ldcg(sp + v0 + 32 * u);
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (v0 + 32 * u < nvec) dp[v0 + 32 * u] = r[u];
            }
            __syncwarp();
            if (lane == 0) red_release_gpu_add(&a.ag_ready[src * ((Tr + 63) / 64) + tl / 64], 1u);
        }
        continue;
    }
    const int claim_end = min(base + CLAIM, nag + total) - nag;
    for (int pq = base - nag; pq < claim_end; ++pq) {
        const int pp = a.row_rot ? (pq + a.row_rot) % total : pq;
        const int i = a.pad_row_tok[pp];
        uint4* d = reinterpret_cast<uint4*>(a.a_dst + (int64_t)pp * K);
        const int ds = (a.dup_src && i >= 0) ? a.dup_src[pp] : -1;
        if (i < 0) {
            for (int v = lane; v < nvec; v += 32) d[v] = make_uint4(0, 0, 0, 0);
        } else if (a.src_bufs8 && ds < 0) {
            // FP8 pull: 16 E4M3 codes per lane-step -> dequantise -> 2 x 16 B bf16
            const int t = i / a.topk;
            const int src = t / a.tokens_per_rank;
            const int tl = t - src * a.tokens_per_rank;
            const uint4* sp = reinterpret_cast<const uint4*>(a.src_bufs8[src] + (int64_t)tl * K);
            const float* sc = a.src_scales[src] + (int64_t)tl * (K / a.src_scale_group);
            const float rs = a.row_scale ? a.row_scale[pp] : 1.0f;
            const int n16 = K / 16;
            constexpr int U8 = 8;
            for (int v0 = lane; v0 < n16; v0 += 32 * U8) {
                uint4 c[U8];
                float f[U8];
#pragma unroll
                for (int q = 0; q < U8; ++q) {
                    const int v = v0 + 32 * q;
                    if (v < n16) {
                        c[q] = sp[v];
                        f[q] = sc[(v * 16) / a.src_scale_group];
                    }
                }
#pragma unroll
                for (int q = 0; q < U8; ++q) {
                    const int v = v0 + 32 * q;
                    if (v < n16) {
                        const float fs = f[q] * rs;
                        const uint32_t w[4] = {c[q].x, c[q].y, c[q].z, c[q].w};
                        uint32_t o[8];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 lo = e4m3x2_to_f32x2((uint16_t)(w[e] & 0xffff));
                            const float2 hi = e4m3x2_to_f32x2((uint16_t)(w[e] >> 16));
                            o[2 * e] = pack_bf16x2(lo.x * fs, lo.y * fs);
                            o[2 * e + 1] = pack_bf16x2(hi.x * fs, hi.y * fs);
                        }
                        d[2 * v] = make_uint4(o[0], o[1], o[2], o[3]);
                        d[2 * v + 1] = make_uint4(o[4], o[5], o[6], o[7]);
                    }
                }
            }
        } else {
            // bf16 row copy in segments (one code path, 16 x 16 B loads in flight
            // per lane = 8 KB per warp):
            //   pull         1 segment: the token row on its owning rank (NVLink)
            //   dedup        1 segment: the token's earlier row ds (< pp) in a_dst,
            //                after it has landed (no wait cycle: ds < pp)
            //   A2A gather   n_src segments of gather_cols columns, own rank first
            const uint4* sp = nullptr;
            float rs = 1.0f;
            int nseg = 1, seg_vec = nvec;
            if (ds >= 0) {
                if (lane == 0) {
                    const uint64_t t0 = globaltimer();
                    while (ld_acquire_gpu(&a.row_done[ds]) == 0u) {
                        if (globaltimer() - t0 > 4000000000ull) {
                            atomicExch(a.err, 2);
                            break;
                        }
                    }
                }
                __syncwarp();
                sp = reinterpret_cast<const uint4*>(a.a_dst + (int64_t)ds * K);
            } else if (a.gather_cols > 0) {
                nseg = a.n_src;
                seg_vec = a.gather_cols / 8;
            } else {
                const int t = i / a.topk;
                const int src = t / a.tokens_per_rank;
                const int tl = t - src * a.tokens_per_rank;
                if (nag > 0 && src != a.self_rank) {
                    // ag_rs: the row was all-gathered into ag_dst by this kernel's comm warps
                    if (lane == 0) {
                        const uint32_t want = (uint32_t)min(64, Tr - (tl / 64) * 64);
                        const uint32_t* flag = &a.ag_ready[src * ((Tr + 63) / 64) + tl / 64];
                        const uint64_t t0 = globaltimer();
                        while (ld_acquire_gpu(flag) < want) {
                            if (globaltimer() - t0 > 4000000000ull) {
                                atomicExch(a.err, 2);
                                break;
                            }
                        }
                    }
                    __syncwarp();
                    sp = reinterpret_cast<const uint4*>(a.ag_dst + (int64_t)t * K);
                } else {
                    sp = reinterpret_cast<const uint4*>(a.src_bufs[src] + (int64_t)tl * K);
                }
                if (a.row_scale) rs = a.row_scale[pp];
            }
            for (int sg = 0; sg < nseg; ++sg) {
                uint4* dp = d;
                if (a.gather_cols > 0) {
                    const int src = (a.src_rot + sg) % a.n_src;
                    sp = reinterpret_cast<const uint4*>(a.src_bufs[src] + (int64_t)(a.src_row0 + i) * a.gather_cols);
                    dp = d + src * seg_vec;
                }
                constexpr int U = 16;
                for (int v0 = lane; v0 < seg_vec; v0 += 32 * U) {
                    uint4 r[U];
#pragma unroll
                    for (int q = 0; q < U; ++q)
                        if (v0 + 32 * q < seg_vec) r[q] = __ldcg(sp + v0 + 32 * q);
                    if (rs != 1.0f) {
#pragma unroll
                        for (int q = 0; q < U; ++q) {
                            const float2 p0 = unpack_bf16x2(r[q].x), p1 = unpack_bf16x2(r[q].y),
                                         p2 = unpack_bf16x2(r[q].z), p3 = unpack_bf16x2(r[q].w);
                            r[q] = make_uint4(pack_bf16x2(p0.x * rs, p0.y * rs), pack_bf16x2(p1.x * rs, p1.y * rs),
                                              pack_bf16x2(p2.x * rs, p2.y * rs), pack_bf16x2(p3.x * rs, p3.y * rs));
                        }
                    }
#pragma unroll
                    for (int q = 0; q < U; ++q)
                        if (v0 + 32 * q < seg_vec) dp[v0 + 32 * q] = r[q];
                }
            }
        }
        __syncwarp();
        if (lane == 0) {
            if (a.row_done && i >= 0) red_release_gpu_add(&a.row_done[pp], 1u);
            fence_proxy_async_global();
            red_release_gpu_add(&a.ready[pp / 128], 1u);
        }
    }
    }
}

template <int BN, int CG, bool A_MN, bool B_MN, bool K_GROUPED, int EPI, bool DISPATCH = false>
__global__ void __launch_bounds__(GemmCfg<BN, CG>::THREADS + (DISPATCH ? 32 * GemmCfg<BN, CG>::COMM_WARPS : 0) +
                                  (EPI == EPI_SCATTER_RS ? 32 : 0), 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const GemmArgs args) {
    using Cfg = GemmCfg<BN, CG>;
    constexpr int BM = Cfg::BM, STAGES = Cfg::STAGES, TILE_M = Cfg::TILE_M;
    constexpr int BN_CTA = Cfg::BN_CTA;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint4* epi_stage = reinterpret_cast<uint4*>(smem + STAGES * Cfg::STAGE_BYTES);
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::EPI_STAGE_BYTES);
    uint64_t* empty_bar = full_bar + STAGES;
    uint64_t* tfull_bar = empty_bar + STAGES;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
    __shared__ int prefix[Cfg::MAX_GROUPS + 1];    // tile prefix per group
    __shared__ int s_rowoff[Cfg::MAX_GROUPS + 1];  // padded row offset per group
    __shared__ int s_kb[Cfg::MAX_GROUPS];          // K-grouped: k blocks per group
    constexpr int QD = 8;                           // tile queue depth
    __shared__ int s_tq[QD];
    __shared__ __align__(8) uint64_t s_tq_full[QD], s_tq_empty[QD];
    // EPI_SCATTER_RS: epilogue warps -> signal warp ring (one entry per tile)
    constexpr int QS = 8;
    __shared__ __align__(8) uint64_t s_sig_full[QS], s_sig_free[QS];
    __shared__ int s_sig_info[QS];

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int G = args.G;
    const int n_tiles = (args.N + BN - 1) / BN;
    const uint32_t cta_rank = CG == 2 ? cluster_ctarank() : 0;
    const bool leader = cta_rank == 0;
    const int unit = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // tile-stride unit
    const int nunits = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;

    // --- setup ---------------------------------------------------------------
    // group tables in shared memory, built by warp 0: every group's row count is
    // loaded in one round trip (lane + 32 j), then a shuffle scan per 32 groups.
    // The roles' per-tile decode reads only shared memory (no global loads on
    // the tile path).
    if (warp == 0) {
        constexpr int NJ = Cfg::MAX_GROUPS / 32;
        int rws[NJ], kr[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int g = lane + 32 * j;
            rws[j] = g < G ? args.group_rows[g] : 0;
            kr[j] = (K_GROUPED && args.group_k_rows && g < G) ? args.group_k_rows[g] : rws[j];
        }
        int carry_t = 0, carry_r = 0;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int g = lane + 32 * j;
            const int rows = rws[j];
            const int tiles = g < G ? (K_GROUPED ? (args.K / TILE_M) * n_tiles
                                                 : ((rows + TILE_M - 1) / TILE_M) * n_tiles)
                                    : 0;
            int it = tiles, ir = rows;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int ut = __shfl_up_sync(0xffffffffu, it, off);
                const int ur = __shfl_up_sync(0xffffffffu, ir, off);
                if (lane >= off) { it += ut; ir += ur; }
            }
            if (g < G) {
                prefix[g] = carry_t + it - tiles;
                s_rowoff[g] = carry_r + ir - rows;
                if (K_GROUPED) s_kb[g] = (kr[j] + 63) >> 6;
            }
            carry_t += __shfl_sync(0xffffffffu, it, 31);
            carry_r += __shfl_sync(0xffffffffu, ir, 31);
        }
        if (lane == 0) {
            prefix[G] = carry_t;
            s_rowoff[G] = carry_r;
        }
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull_bar[a], 1);
            mbar_init(&tempty_bar[a], Cfg::EPI_WARPS * CG);
        }
        // queue consumers: MMA + epilogue warps of the leader, producer +
        // epilogue warps of the peer
        for (int q = 0; q < QD; ++q) {
            mbar_init(&s_tq_full[q], 1);
            mbar_init(&s_tq_empty[q], (1 + Cfg::EPI_WARPS) * CG);
        }
        if (EPI == EPI_SCATTER_RS)
            for (int q = 0; q < QS; ++q) {
                mbar_init(&s_sig_full[q], Cfg::EPI_WARPS);
                mbar_init(&s_sig_free[q], 1);
            }
        fence_barrier_init();
    }
    if (warp == 1) {
        if (CG == 2) tmem_alloc_2sm<Cfg::TMEM_COLS>(tmem_slot);
        else tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int total_tiles = prefix[G] + (K_GROUPED ? 0 : args.split_last);
    // dynamic for M-grouped GEMMs (M = 128 tail tiles and dispatch waits make
    // tile costs uneven, and a drifting static stride breaks the L2 sharing of
    // weight panels: 2.3x DRAM reads measured); the K-grouped wgrads keep the
    // static stride, which measured faster for them
    // long-K M-grouped GEMMs (K >= 8192: the Mixtral fc2 / fc1 dgrad) keep the
    // single-lane issue and the static stride: there the faster warp-convergent
    // issue and the dynamic schedule raised DRAM re-reads (fc1 dgrad: 3.0 GB ->
    // 5.2 / 8.5 GB, ncu) and, under the power cap, the time
    const bool legacy = !K_GROUPED && args.K >= 8192 && G > 1;   // single-group GEMMs have no tails to drift on
    const bool dyn = !K_GROUPED && !legacy && args.tile_counter != nullptr;
    // i-th tile of this CTA (pair): static stride, or dynamic. The leader's
    // producer fetches (atomic, in order) and publishes to the local queue and,
    // for a pair, to the peer's; every other role dequeues. -1 ends the loop.
    // The producer claims a tile only when it starts loading it (LA = 0): the
    // tiles in flight across the grid then form one contiguous window of the
    // tile order, so concurrent tiles share their weight / activation panels in
    // L2. (Claiming ahead spreads each CTA's next claims over several waves and
    // doubled the DRAM reads of the Mixtral fc1-dgrad.) The next atomic is
    // always in flight; the peer CTA learns the tile while the MMA still works
    // through the 6 staged k-blocks of the previous one.
    constexpr int LA = 0;   // < QD: the producer's own slot is never overwritten
    int t_ahead = (dyn && warp == 0 && lane == 0 && leader) ? atomicAdd(args.tile_counter, 1) : 0;
    int published = 0;
    bool ended = false;
    auto fetch_tile = [&](int i) -> int {
        if (!dyn) return unit + i * nunits < total_tiles ? unit + i * nunits : -1;
        while (!ended && published <= i + LA) {
            const int slot = published % QD;
            const uint32_t ph = (uint32_t)(published / QD) & 1u;
            int t = 0;
            if (lane == 0) {
                t = t_ahead;
                if (t >= total_tiles) t = -1;
                else t_ahead = atomicAdd(args.tile_counter, 1);
                mbar_wait(&s_tq_empty[slot], ph ^ 1u);
                s_tq[slot] = t;
                if (CG == 2) {
                    st_shared_cluster(map_to_cta(&s_tq[slot], 1), t);
                    mbar_arrive_release_cluster(map_to_cta(&s_tq_full[slot], 1));
                }
                mbar_arrive(&s_tq_full[slot]);
            }
            t = __shfl_sync(0xffffffffu, t, 0);
            ended = t < 0;
            ++published;
        }
        // this CTA wrote slot i itself (published > i)
        return *reinterpret_cast<volatile int*>(&s_tq[i % QD]);
    };
    auto next_tile = [&](int i) -> int {
        if (!dyn) return unit + i * nunits < total_tiles ? unit + i * nunits : -1;
        const int slot = i % QD;
        const uint32_t ph = (uint32_t)(i / QD) & 1u;
        int t = 0;
        if (lane == 0) {
            while (!mbar_try_wait_cluster(&s_tq_full[slot], ph)) {
            }
            t = *reinterpret_cast<volatile int*>(&s_tq[slot]);
            if (CG == 2 && !leader) mbar_arrive_release_cluster(map_to_cta(&s_tq_empty[slot], 0));
            else mbar_arrive(&s_tq_empty[slot]);
        }
        return __shfl_sync(0xffffffffu, t, 0);
    };

    if (warp == 0) {
        // ===================== TMA producer =====================
        // CONV: whole warp in convergence, one elected lane issues (as for the
        // MMA); otherwise lane 0 alone (long-K GEMMs, see `legacy`)
        auto producer = [&](auto conv_tag) {
            constexpr bool CONV = decltype(conv_tag)::value;
            int stage = 0;
            uint32_t phase = 0;
            const int arow = (int)cta_rank * BM;       // this CTA's A rows within the tile
            const int bcol = (int)cta_rank * BN_CTA;   // this CTA's B rows/cols within the tile
            for (int it = 0;; ++it) {
                const int t = leader ? fetch_tile(it) : next_tile(it);
                if (t < 0) break;
                const TileInfo ti = decode_tile<TILE_M, K_GROUPED>(t, prefix, s_rowoff, s_kb, args, G, n_tiles);
                for (int kb = 0; kb < ti.kblocks; ++kb) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
                    uint8_t* sb = sa + Cfg::A_BYTES;
                    uint64_t* fb = &full_bar[stage];
                    uint32_t fb_leader = 0;
                    if (CG == 2) {
                        fb_leader = map_to_cta(fb, 0);
                        if (leader) {
                            if (CONV) mbar_arrive_expect_tx_warp(fb, CG * Cfg::STAGE_BYTES);
                            else mbar_arrive_expect_tx(fb, CG * Cfg::STAGE_BYTES);
                        }
                    } else {
                        if (CONV) mbar_arrive_expect_tx_warp(fb, Cfg::STAGE_BYTES);
                        else mbar_arrive_expect_tx(fb, Cfg::STAGE_BYTES);
                    }
                    auto load = [&](void* dst, const CUtensorMap* map, int c0, int c1) {
                        if (CONV) {
                            if (CG == 2) tma_load_2d_2sm_warp(dst, map, fb_leader, c0, c1);
                            else tma_load_2d_warp(dst, map, fb, c0, c1);
                        } else {
                            if (CG == 2) tma_load_2d_2sm(dst, map, fb_leader, c0, c1);
                            else tma_load_2d(dst, map, fb, c0, c1);
                        }
                    };
                    if (!K_GROUPED) {
                        if (DISPATCH && kb == 0) {
                            // wait until this tile's permuted rows (one counter per
                            // 128-row block) have landed
                            const uint32_t* rdy = &args.ready[ti.row0 / BM];
                            const int nblk = ti.half_tile ? 1 : CG;
                            if (lane == 0) {
                                const uint64_t t0 = globaltimer();
                                for (int b = 0; b < nblk; ++b)
                                    while (ld_acquire_gpu(rdy + b) < (uint32_t)BM) {
                                        if (globaltimer() - t0 > 4000000000ull) {
                                            atomicExch(args.err, 2);
                                            break;
                                        }
                                    }
                            }
                            if (CONV) __syncwarp();
                            fence_proxy_async_global();   // every lane: the issuing lane is elected
                        }
                        // half tile: each CTA of the pair takes 64 rows (the box's other
                        // 64 rows are loaded but not read by the M = 128 UMMA)
                        load(sa, &tmA, kb * 64, ti.row0 + (ti.half_tile ? (int)cta_rank * 64 : arow));
                        if (!B_MN) {
                            const int bbr = args.b_box_rows > 0 ? args.b_box_rows : BN_CTA;
                            for (int j = 0; j < BN_CTA; j += bbr)
                                load(sb + j * 128, &tmB, kb * 64,
                                     ti.g * args.b_group_stride + ti.n * BN + bcol + j);
                        } else {
#pragma unroll
                            for (int j = 0; j < BN_CTA / 64; ++j)
                                load(sb + j * 8192, &tmB, ti.n * BN + bcol + j * 64,
                                     ti.g * args.b_group_stride + kb * 64);
                        }
                    } else {
                        // wgrad: A = [rows, M] MN-major, B = [rows, N] MN-major
#pragma unroll
                        for (int j = 0; j < BM / 64; ++j)
                            load(sa + j * 8192, &tmA, ti.m * TILE_M + arow + j * 64, ti.row0 + kb * 64);
#pragma unroll
                        for (int j = 0; j < BN_CTA / 64; ++j)
                            load(sb + j * 8192, &tmB, ti.n * BN + bcol + j * 64, ti.row0 + kb * 64);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        };
        if (legacy) {
            if (lane == 0) producer(std::false_type{});
        } else {
            producer(std::true_type{});
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA) =====================
        // The whole warp walks the tile / k-block sequence in convergence, so
        // descriptors and TMEM addresses stay warp-uniform (uniform registers)
        // and one elected lane issues: no per-MMA register broadcast loops.
        auto mma_role = [&](auto conv_tag) {
            constexpr bool CONV = decltype(conv_tag)::value;
            constexpr uint32_t idesc_full = make_idesc(TILE_M, BN, 1, A_MN, B_MN);
            constexpr uint32_t idesc_half = make_idesc(128, BN, 1, A_MN, B_MN);
            // stage s's descriptors = stage 0's + s * STAGE_BYTES / 16 (14-bit
            // address field, smem < 256 KB); k step within a stage: +32 B
            // (K-major) or +2048 B (MN-major), i.e. +2 / +128 in 16-byte units
            const uint32_t s0 = smem_u32(smem);
            const uint64_t a_base = A_MN ? make_sdesc(s0, 8192, 1024) : make_sdesc(s0, 16, 1024);
            const uint64_t b_base = B_MN ? make_sdesc(s0 + Cfg::A_BYTES, 8192, 1024)
                                         : make_sdesc(s0 + Cfg::A_BYTES, 16, 1024);
            constexpr uint64_t a_kstep = A_MN ? 128 : 2, b_kstep = B_MN ? 128 : 2;
            constexpr uint64_t stage_step = Cfg::STAGE_BYTES >> 4;
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int it = 0;; ++it) {
                const int t = next_tile(it);
                if (t < 0) break;
                const TileInfo ti = decode_tile<TILE_M, K_GROUPED>(t, prefix, s_rowoff, s_kb, args, G, n_tiles);
                if (ti.kblocks == 0) continue;
                mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                const uint32_t idesc = ti.half_tile ? idesc_half : idesc_full;
                for (int kb = 0; kb < ti.kblocks; ++kb) {
                    mbar_wait(&full_bar[stage], phase);
                    tc_fence_after();
                    const uint64_t ad0 = a_base + (uint64_t)stage * stage_step;
                    const uint64_t bd0 = b_base + (uint64_t)stage * stage_step;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t ad = ad0 + kk * a_kstep, bd = bd0 + kk * b_kstep;
                        if (CONV) {
                            if (CG == 2) umma_bf16_2sm_warp(d_tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
                            else umma_bf16_warp(d_tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
                        } else {
                            if (CG == 2) umma_bf16_2sm(d_tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
                            else umma_bf16(d_tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
                        }
                    }
                    if (CONV) {
                        if (CG == 2) umma_commit_2sm_mc_warp(&empty_bar[stage]);
                        else umma_commit_warp(&empty_bar[stage]);
                    } else {
                        if (CG == 2) umma_commit_2sm_mc(&empty_bar[stage]);
                        else umma_commit(&empty_bar[stage]);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                if (CONV) {
                    if (CG == 2) umma_commit_2sm_mc_warp(&tfull_bar[acc]);
                    else umma_commit_warp(&tfull_bar[acc]);
                } else {
                    if (CG == 2) umma_commit_2sm_mc(&tfull_bar[acc]);
                    else umma_commit(&tfull_bar[acc]);
                }
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        };
        if (leader) {
            if (legacy) {
                if (lane == 0) mma_role(std::false_type{});
            } else {
                mma_role(std::true_type{});
            }
        }
    } else if (EPI == EPI_SCATTER_RS && warp == 2 + Cfg::EPI_WARPS) {
        // ===================== GEMM-RS signal warp =====================
        // Announces this CTA's part of each peer-owned tile once its 8 epilogue
        // warps stored it: the CTA-scope mbarrier orders their NVLink stores
        // before this lane's system-scope release, so the epilogue warps never
        // wait for the link to drain.
        // Entries that completed while a fence drained are announced together
        // behind one fence (one link drain per batch, not per tile).
        if (lane == 0) {
            bool done = false;
            for (int sq = 0; !done;) {
                mbar_wait(&s_sig_full[sq % QS], (uint32_t)(sq / QS) & 1u);
                int end = sq + 1;
                while (end - sq < QS && mbar_try_wait(&s_sig_full[end % QS], (uint32_t)(end / QS) & 1u)) ++end;
                fence_acq_rel_sys();
                for (int q = sq; q < end; ++q) {
                    const int info = *reinterpret_cast<volatile int*>(&s_sig_info[q % QS]);
                    if (info >= 0)
                        red_relaxed_sys_add(args.rs_cnt[info >> 24] + (info & 0xffffff), (uint32_t)Cfg::EPI_WARPS);
                    if (info == -2) done = true;
                    mbar_arrive(&s_sig_free[q % QS]);
                }
                sq = end;
            }
        }
    } else if (DISPATCH && warp >= 2 + Cfg::EPI_WARPS) {
        // ===================== dispatch (comm warps) =====================
        dispatch_warp<TILE_M>(args, args.K, lane);
    } else {
        // ===================== epilogue (warps 2..9) =====================
        const int ew = warp - 2;
        const int quarter = warp & 3;           // TMEM lane quarter this warp may access
        const int half = ew >> 2;               // column half
        const int r_in_cta = quarter * 32 + lane;
        const uint32_t tempty_leader = CG == 2 ? map_to_cta(&tempty_bar[0], 0) : 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        int sig_sq = 0;
        // EPI_SCATTER_RS: publish one ring entry per tile (warp 0 of the epilogue
        // writes it once the signal warp freed the slot; all 8 warps arrive after
        // their stores, which orders those stores before the signal warp's release)
        auto rs_sig = [&](int sq, int info) {
            const int slot = sq % QS;
            __syncwarp();
            if (lane == 0) {
                if (ew == 0) {
                    mbar_wait(&s_sig_free[slot], ((uint32_t)(sq / QS) & 1u) ^ 1u);
                    s_sig_info[slot] = info;
                }
                mbar_arrive(&s_sig_full[slot]);
            }
        };
        for (int it = 0;; ++it) {
            const int t = next_tile(it);
            if (t < 0) {
                if (EPI == EPI_SCATTER_RS) rs_sig(sig_sq, -2);
                break;
            }
            const TileInfo ti = decode_tile<TILE_M, K_GROUPED>(t, prefix, s_rowoff, s_kb, args, G, n_tiles);
            const int n0 = ti.n * BN;
            int64_t orow;
            if (K_GROUPED) {
                int mi = ti.m * TILE_M + (int)cta_rank * BM + r_in_cta;
                if (args.interleave_rows) {
                    const int blk = mi >> 7, w = mi & 127;
                    mi = w < 64 ? blk * 64 + w : (args.K >> 1) + blk * 64 + (w - 64);
                }
                orow = (int64_t)ti.g * args.K + mi;
            } else if (ti.half_tile) {
                // M = 128 pair tile: each CTA holds 64 rows; TMEM lanes 0-63 carry
                // accumulator columns [0, BN/2), lanes 64-127 columns [BN/2, BN),
                // both in TMEM columns [0, BN/2) (scripts/probe_tmem_layout.cu)
                orow = (int64_t)ti.row0 + (int)cta_rank * 64 + (quarter & 1) * 32 + lane;
            } else {
                orow = (int64_t)ti.row0 + (int)cta_rank * BM + r_in_cta;
            }
            if (ti.kblocks == 0) {
                // empty contraction (expert received no rows): D = 0
                const int c_lo = half * (BN / 2);
                if (EPI == EPI_STORE_BF16) {
                    uint16_t* o = reinterpret_cast<uint16_t*>(args.out) + orow * args.ldo + n0;
                    for (int c = c_lo; c < c_lo + BN / 2; c += 8)
                        if (n0 + c < args.N) *reinterpret_cast<uint4*>(o + c) = make_uint4(0, 0, 0, 0);
                } else if (EPI == EPI_STORE_F32) {
                    float* o = reinterpret_cast<float*>(args.out) + orow * args.ldo + n0;
                    for (int c = c_lo; c < c_lo + BN / 2; c += 4)
                        if (n0 + c < args.N) *reinterpret_cast<float4*>(o + c) = make_float4(0, 0, 0, 0);
                }
                continue;
            }
            // half tile: one warp per lane quarter covers the quarter's BN/2 columns
            const int ch = ti.half_tile ? (quarter >> 1) : half;
            const bool active = !ti.half_tile || half == 0;
            uint4 va[4], vb[4];
            if constexpr (EPI == EPI_SWIGLU_BWD) {
                // the epilogue's own global operand (fc1_out) does not depend on the
                // accumulator: put the first chunk in flight before waiting for it
                if (active) {
                    const int j = n0 + ch * (BN / 2);
                    const int ia = (j >> 6) * 128 + (j & 63);
                    const uint16_t* f1 = args.aux + orow * args.ld_aux;
                    load_rows32_issue(va, f1 + ia, lane);
                    load_rows32_issue(vb, f1 + ia + 64, lane);
                }
            }
            mbar_wait(&tfull_bar[acc], acc_phase);
            tc_fence_after();
            const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
            if (active)
                epilogue_rows<BN, EPI, K_GROUPED>(args, ti, orow, tbase, ch * (BN / 2), ch, n_tiles,
                                                  epi_stage + ew * 128, ti.half_tile ? ch * (BN / 2) : 0, va, vb);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 2) mbar_arrive_cluster(tempty_leader + acc * 8);
                else mbar_arrive(&tempty_bar[acc]);
            }
            if constexpr (EPI == EPI_SCATTER_RS) {
                // hand the tile to the signal warp (peer-owned: owner and tile index)
                const int owner = ti.row0 / args.rs_rows;
                const int info = owner != args.self_rank
                                     ? (owner << 24) | ((ti.m - owner * (args.rs_rows / TILE_M)) * n_tiles + ti.n)
                                     : -1;
                rs_sig(sig_sq++, info);
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }

    __syncwarp();
    __syncthreads();
    if (CG == 2) cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        if (CG == 2) tmem_dealloc_2sm<Cfg::TMEM_COLS>(tmem_base);
        else tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
    }
}

}  // namespace moe
