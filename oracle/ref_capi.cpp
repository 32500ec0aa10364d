// ref_capi.cpp — a flat C ABI over the REFERENCE's own routing and numerics
// code (/root/reference/proj/core/src/{routing,numerics}.cpp, compiled
// unmodified from where they lie by oracle/Makefile into oracle/_ref/).
//
// TEST INFRASTRUCTURE ONLY: used to pin the oracle restatement
// (moe_oracle.c), to generate tests/golden/ fixtures, and as the
// `--impl reference` CPU arm of bench.py. The product never links it.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "moeplan/numerics.hpp"
#include "moeplan/routing.hpp"

using namespace moeplan;

namespace {
int status_of(const std::exception& e) {
    return dynamic_cast<const std::domain_error*>(&e) ? -2 : -1;
}

routing::RoutingAssignment make_assignment(int64_t T, int64_t E, int64_t k, int64_t n_groups,
                                           const int32_t* experts, const int32_t* src,
                                           const uint8_t* dropped) {
    routing::RoutingAssignment a;
    a.num_experts = E;
    a.top_k = k;
    a.n_groups = n_groups;
    a.experts.resize(T);
    a.source_rank.resize(T);
    a.dropped.resize(T);
    for (int64_t t = 0; t < T; ++t) {
        a.experts[t].assign(experts + t * k, experts + (t + 1) * k);
        a.source_rank[t] = src[t];
        a.dropped[t] = static_cast<char>(dropped[t]);
    }
    return a;
}
}  // namespace

extern "C" {

// routing.hpp:49-55. mode: 0 uniform, 1 random, 2 skewed.
int ref_simulate_routing(int64_t T, int64_t E, int64_t k, int mode, uint64_t seed,
                         double zipf_s, double cf, int64_t n_groups, int32_t* experts,
                         int32_t* source_rank, uint8_t* dropped) {
    try {
        routing::RoutingSpec spec;
        spec.mode = static_cast<routing::RoutingMode>(mode);
        spec.seed = seed;
        spec.zipf_s = zipf_s;
        const auto a = routing::simulate_routing(T, E, k, spec, cf, n_groups);
        for (int64_t t = 0; t < T; ++t) {
            for (int64_t j = 0; j < k; ++j) experts[t * k + j] = a.experts[t][j];
            source_rank[t] = a.source_rank[t];
            dropped[t] = static_cast<uint8_t>(a.dropped[t]);
        }
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// routing.hpp:72. Returns rows (>= 0) or a negative status.
int64_t ref_build_scatter_map(int64_t T, int64_t E, int64_t k, int64_t n_groups,
                              const int32_t* experts, const int32_t* src,
                              const uint8_t* dropped, int64_t n, int64_t my_rank,
                              int64_t* row_map_in, int64_t* row_map_out, int64_t* inverse_map,
                              int64_t* per_expert_counts, int32_t* out_expert,
                              int32_t* out_source_rank) {
    try {
        const auto a = make_assignment(T, E, k, n_groups, experts, src, dropped);
        const auto m = routing::build_scatter_map(a, n, my_rank);
        for (int64_t r = 0; r < m.rows; ++r) {
            row_map_in[r] = m.row_map_in[r];
            row_map_out[r] = m.row_map_out[r];
            inverse_map[r] = m.inverse_map[r];
            out_expert[r] = m.out_expert[r];
            out_source_rank[r] = m.out_source_rank[r];
        }
        for (int64_t e = 0; e < E; ++e) per_expert_counts[e] = m.per_expert_counts[e];
        return m.rows;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// routing.hpp:88-89. Dependent ranks returned as a bitmask per tile.
int64_t ref_sort_tokens_for_tiles(int64_t T, int64_t E, int64_t k, int64_t n_groups,
                                  const int32_t* experts, const int32_t* src,
                                  const uint8_t* dropped, int64_t n, int64_t my_rank,
                                  int64_t tile_rows, int32_t* tile_expert, int64_t* tile_begin,
                                  int64_t* tile_end, uint64_t* tile_rank_mask,
                                  int32_t* tile_rank_lo, int32_t* tile_rank_hi) {
    try {
        const auto a = make_assignment(T, E, k, n_groups, experts, src, dropped);
        const auto m = routing::build_scatter_map(a, n, my_rank);
        const auto lay = routing::sort_tokens_for_tiles(m, a, tile_rows);
        for (size_t i = 0; i < lay.tiles.size(); ++i) {
            const auto& t = lay.tiles[i];
            tile_expert[i] = t.expert;
            tile_begin[i] = t.row_begin;
            tile_end[i] = t.row_end;
            uint64_t mask = 0;
            for (int r : t.dependent_ranks) mask |= 1ull << r;
            tile_rank_mask[i] = mask;
            tile_rank_lo[i] = t.dependent_ranks.front();
            tile_rank_hi[i] = t.dependent_ranks.back();
        }
        return static_cast<int64_t>(lay.tiles.size());
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// routing.hpp:101.
int ref_balance_metrics(int64_t T, int64_t E, int64_t k, int64_t n_groups,
                        const int32_t* experts, const int32_t* src, const uint8_t* dropped,
                        int64_t n, int64_t* per_group_load, double* loss, int64_t* capacity,
                        double* drop_rate) {
    try {
        const auto a = make_assignment(T, E, k, n_groups, experts, src, dropped);
        const auto s = routing::balance_metrics(a, n);
        for (int64_t g = 0; g < n; ++g) per_group_load[g] = s.per_group_load[g];
        *loss = s.balance_loss_value;
        *capacity = s.capacity;
        *drop_rate = s.drop_rate;
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// numerics.hpp:31. fmt: 0 fp32, 1 bf16, 2 fp8_e4m3.
void ref_round_to(int fmt, const double* x, int64_t count, double* out) {
    for (int64_t i = 0; i < count; ++i)
        out[i] = numerics::round_to(static_cast<Format>(fmt), x[i]);
}

// numerics.hpp:61-62. gran: 0 per_tensor, 1 per_token, 2 per_channel, 3 grouped.
int ref_quantize(const double* x, int64_t rows, int64_t cols, int gran, int64_t group_size,
                 int fmt, double* codes, double* scales, int64_t* num_blocks) {
    try {
        numerics::QuantScheme s;
        s.granularity = static_cast<numerics::Granularity>(gran);
        s.group_size = group_size;
        std::vector<double> v(x, x + rows * cols);
        const auto q = numerics::quantize(v, rows, cols, s, static_cast<Format>(fmt));
        std::memcpy(codes, q.codes.data(), sizeof(double) * q.codes.size());
        std::memcpy(scales, q.scales.data(), sizeof(double) * q.scales.size());
        *num_blocks = static_cast<int64_t>(q.scales.size());
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// numerics.hpp:77-78. kind: 0 ring_bf16, 1 a2a_fp32.
int ref_emulate_reduce(const double* vectors, int64_t ranks, int64_t dim, int kind,
                       double* out) {
    try {
        std::vector<std::vector<double>> v(ranks);
        for (int64_t r = 0; r < ranks; ++r) v[r].assign(vectors + r * dim, vectors + (r + 1) * dim);
        const auto o = numerics::emulate_reduce(v, static_cast<numerics::ReduceKind>(kind));
        std::memcpy(out, o.data(), sizeof(double) * o.size());
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// Timing of the reference's own calls with the value types built once outside
// the timed region (bench.py cpu_baseline; the reference's bench does the
// same list, bench_moeplan.cpp:128-170). Median of `reps` single-threaded runs.
// ms[0] build_scatter_map x n, ms[1] sort_tokens_for_tiles(tile_rows) x n on
// those maps, ms[2] balance_metrics.
int ref_time_routing(int64_t T, int64_t E, int64_t k, int64_t n_groups, const int32_t* experts,
                     const int32_t* src, const uint8_t* dropped, int64_t n, int64_t tile_rows,
                     int reps, double* ms) {
    try {
        using clk = std::chrono::steady_clock;
        const auto a = make_assignment(T, E, k, n_groups, experts, src, dropped);
        std::vector<double> t0s, t1s, t2s;
        for (int it = 0; it < reps; ++it) {
            std::vector<routing::ScatterMap> maps;
            auto c0 = clk::now();
            for (int64_t r = 0; r < n; ++r) maps.push_back(routing::build_scatter_map(a, n, r));
            auto c1 = clk::now();
            size_t tiles = 0;
            for (int64_t r = 0; r < n; ++r) tiles += routing::sort_tokens_for_tiles(maps[r], a, tile_rows).tiles.size();
            auto c2 = clk::now();
            const auto st = routing::balance_metrics(a, n);
            auto c3 = clk::now();
            if (tiles == 0 && st.capacity < 0) return -1;  // keep the results live
            t0s.push_back(std::chrono::duration<double, std::milli>(c1 - c0).count());
            t1s.push_back(std::chrono::duration<double, std::milli>(c2 - c1).count());
            t2s.push_back(std::chrono::duration<double, std::milli>(c3 - c2).count());
        }
        auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
        ms[0] = med(t0s);
        ms[1] = med(t1s);
        ms[2] = med(t2s);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// ms[0] quantize(x, rows, cols, gran) in fmt; ms[1] emulate_reduce(vectors, kind)
int ref_time_numerics(const double* x, int64_t rows, int64_t cols, int gran, int64_t group_size,
                      int fmt, const double* vectors, int64_t ranks, int64_t dim, int kind, double* ms) {
    try {
        using clk = std::chrono::steady_clock;
        numerics::QuantScheme s;
        s.granularity = static_cast<numerics::Granularity>(gran);
        s.group_size = group_size;
        std::vector<double> v(x, x + rows * cols);
        std::vector<std::vector<double>> vv(ranks);
        for (int64_t r = 0; r < ranks; ++r) vv[r].assign(vectors + r * dim, vectors + (r + 1) * dim);
        auto c0 = clk::now();
        const auto q = numerics::quantize(v, rows, cols, s, static_cast<Format>(fmt));
        auto c1 = clk::now();
        const auto o = numerics::emulate_reduce(vv, static_cast<numerics::ReduceKind>(kind));
        auto c2 = clk::now();
        if (q.scales.empty() || o.empty()) return -1;
        ms[0] = std::chrono::duration<double, std::milli>(c1 - c0).count();
        ms[1] = std::chrono::duration<double, std::milli>(c2 - c1).count();
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

}  // extern "C"
