// moeplan_compat.cpp — drop-in implementation of the reference's routing
// interface (/root/reference/proj/core/include/moeplan/routing.hpp) on top of
// the C ABI of libmoe_b200.so. A MoEPlan build links this library instead of
// core/src/routing.cpp and every caller keeps its code: the maps are computed
// by the sm_100a kernels (capacity drop, stable permutation, tile layout,
// balance counts) and copied back into the reference's value types.
//
// Built against the reference's own header (the types must be identical);
// see INTEGRATION.md. Synchronous, like the functions it replaces.
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nlohmann/json.hpp>

#include "moeplan/routing.hpp"
#include "../../include/moe_b200.h"

namespace {

void require(bool cond, const char* msg) {
    if (!cond) throw std::domain_error(msg);
}

// Map a C-ABI status onto the reference's exception split.
void check(moe_status st) {
    if (st == MOE_OK) return;
    if (st == MOE_ERR_INVALID) throw std::domain_error(moe_last_error());
    throw std::runtime_error(std::string("moe_b200: ") + moe_last_error());
}

void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(size_t n) { cuda(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void upload(const std::vector<T>& h) {
        if (!h.empty()) cuda(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    }
    std::vector<T> download(size_t n) const {
        std::vector<T> h(n);
        if (n) cuda(cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost));
        return h;
    }
};

struct DeviceAssignment {
    DevBuf<int32_t> experts, src;
    DevBuf<uint8_t> dropped;
    explicit DeviceAssignment(const moeplan::routing::RoutingAssignment& a)
        : experts(a.tokens() * a.top_k), src(a.tokens()), dropped(a.tokens()) {
        const long long T = a.tokens();
        std::vector<int32_t> ex(T * a.top_k);
        for (long long t = 0; t < T; ++t) {
            if ((long long)a.experts[t].size() != a.top_k)
                throw std::domain_error("every token needs top_k expert ids");
            for (long long j = 0; j < a.top_k; ++j) ex[t * a.top_k + j] = a.experts[t][j];
        }
        experts.upload(ex);
        src.upload(std::vector<int32_t>(a.source_rank.begin(), a.source_rank.end()));
        dropped.upload(std::vector<uint8_t>(a.dropped.begin(), a.dropped.end()));
    }
};

int32_t max_source_rank(const moeplan::routing::RoutingAssignment& a) {
    int32_t m = 0;
    for (int r : a.source_rank) m = std::max(m, r);
    return m;
}

}  // namespace

namespace moeplan::routing {

long long RoutingAssignment::retained_slots() const {
    long long slots = 0;
    for (size_t t = 0; t < experts.size(); ++t)
        if (!dropped[t]) slots += static_cast<long long>(experts[t].size());
    return slots;
}

int RoutingAssignment::group_of_expert(int expert) const {
    return static_cast<int>(expert / (num_experts / n_groups));
}

// Synthetic assignment generator (host: libstdc++ distributions are part of
// its contract) + the capacity drop on the GPU.
RoutingAssignment simulate_routing(long long tokens, long long num_experts, long long top_k,
                                   const RoutingSpec& spec, double capacity_factor,
                                   long long n_groups) {
    require(tokens >= 0, "tokens must be >= 0");
    require(num_experts >= 1 && top_k >= 1, "counts must be >= 1");
    require(top_k <= num_experts, "top_k must not exceed num_experts");
    require(n_groups >= 1, "n_groups must be >= 1");
    require(num_experts % n_groups == 0, "num_experts must divide evenly across groups");
    require(capacity_factor > 0.0, "capacity_factor must be > 0");
    if (spec.mode == RoutingMode::skewed) require(spec.zipf_s >= 0.0, "zipf_s must be >= 0");

    RoutingAssignment a;
    a.num_experts = num_experts;
    a.top_k = top_k;
    a.n_groups = n_groups;
    a.experts.assign(tokens, {});
    a.source_rank.assign(tokens, 0);
    a.dropped.assign(tokens, 0);
    std::mt19937_64 gen(spec.seed);
    std::vector<double> zipf;
    if (spec.mode == RoutingMode::skewed)
        for (long long e = 0; e < num_experts; ++e) zipf.push_back(std::pow(double(e + 1), -spec.zipf_s));
    std::vector<int> ids(num_experts);
    for (long long t = 0; t < tokens; ++t) {
        a.source_rank[t] = static_cast<int>(t * n_groups / std::max<long long>(tokens, 1));
        std::vector<int>& pick = a.experts[t];
        if (spec.mode == RoutingMode::uniform) {
            for (long long j = 0; j < top_k; ++j) pick.push_back(int((t * top_k + j) % num_experts));
        } else if (spec.mode == RoutingMode::random) {
            std::iota(ids.begin(), ids.end(), 0);
            for (long long j = 0; j < top_k; ++j) {
                std::uniform_int_distribution<long long> u(j, num_experts - 1);
                std::swap(ids[j], ids[u(gen)]);
                pick.push_back(ids[j]);
            }
        } else {
            std::vector<double> w = zipf;
            for (long long j = 0; j < top_k; ++j) {
                std::discrete_distribution<int> d(w.begin(), w.end());
                const int e = d(gen);
                pick.push_back(e);
                w[e] = 0.0;
            }
        }
    }
    if (tokens > 0) {
        DeviceAssignment d(a);
        DevBuf<uint8_t> drop(tokens);
        check(moe_capacity_drop(d.experts.p, tokens, num_experts, top_k, n_groups, capacity_factor,
                                drop.p, nullptr));
        const auto h = drop.download(tokens);
        for (long long t = 0; t < tokens; ++t) a.dropped[t] = static_cast<char>(h[t]);
    }
    return a;
}

ScatterMap build_scatter_map(const RoutingAssignment& a, long long n, long long my_rank) {
    require(n >= 1, "n must be >= 1");
    require(my_rank >= 0 && my_rank < n, "my_rank out of range");
    require(a.num_experts % n == 0, "num_experts must be divisible by n");
    const long long T = a.tokens(), k = a.top_k, E = a.num_experts;
    const long long n_src = std::max<long long>(max_source_rank(a) + 1, 1);
    DeviceAssignment d(a);
    const size_t cap = std::max<long long>(T * k, 1);
    DevBuf<int32_t> rmi(cap), cnt(E), oe(cap), osr(cap), offs(E / n + 1), rows(1);
    DevBuf<uint8_t> ws(moe_permute_workspace_size(T, E, k, n_src));
    check(moe_permute(d.experts.p, d.src.p, d.dropped.p, T, E, k, n, my_rank, n_src, rmi.p, cnt.p,
                      oe.p, osr.p, offs.p, rows.p, ws.p, nullptr));
    const int32_t r = rows.download(1)[0];
    ScatterMap m;
    m.my_rank = my_rank;
    m.rows = r;
    const auto in = rmi.download(r);
    const auto ex = oe.download(r);
    const auto sr = osr.download(r);
    const auto c = cnt.download(E);
    m.row_map_in.assign(in.begin(), in.end());
    m.row_map_out.resize(r);
    std::iota(m.row_map_out.begin(), m.row_map_out.end(), 0ll);
    m.inverse_map = m.row_map_in;
    m.per_expert_counts.assign(c.begin(), c.end());
    m.out_expert.assign(ex.begin(), ex.end());
    m.out_source_rank.assign(sr.begin(), sr.end());
    return m;
}

TileLayout sort_tokens_for_tiles(const ScatterMap& map, const RoutingAssignment& a,
                                 long long tile_rows) {
    (void)a;
    require(tile_rows >= 1, "tile_rows must be >= 1");
    TileLayout lay;
    lay.tile_rows = tile_rows;
    if (map.rows == 0) return lay;
    // expert segment offsets over the contiguous expert range present
    const int first = map.out_expert.front(), last = map.out_expert.back();
    std::vector<int32_t> offs(last - first + 2, 0);
    for (int e : map.out_expert) offs[e - first + 1]++;
    for (size_t i = 1; i < offs.size(); ++i) offs[i] += offs[i - 1];
    DevBuf<int32_t> d_src(map.rows), d_off(offs.size());
    d_src.upload(std::vector<int32_t>(map.out_source_rank.begin(), map.out_source_rank.end()));
    d_off.upload(offs);
    const size_t cap = map.rows + offs.size();
    DevBuf<int32_t> te(cap), tb(cap), tend(cap), nt(1);
    DevBuf<uint64_t> tm(cap);
    check(moe_tile_layout(d_src.p, d_off.p, last - first + 1, first, tile_rows, te.p, tb.p, tend.p,
                          tm.p, nt.p, nullptr));
    const int32_t ntiles = nt.download(1)[0];
    const auto he = te.download(ntiles), hb = tb.download(ntiles), hend = tend.download(ntiles);
    const auto hm = tm.download(ntiles);
    for (int32_t i = 0; i < ntiles; ++i) {
        Tile t;
        t.expert = he[i];
        t.row_begin = hb[i];
        t.row_end = hend[i];
        for (int r = 0; r < 64; ++r)
            if ((hm[i] >> r) & 1ull) t.dependent_ranks.push_back(r);
        lay.tiles.push_back(std::move(t));
    }
    return lay;
}

BalanceStats balance_metrics(const RoutingAssignment& a, long long n) {
    require(n >= 1, "n must be >= 1");
    require(a.n_groups == n || a.num_experts % n == 0, "incompatible group count");
    BalanceStats s;
    s.per_group_load.assign(n, 0);
    const long long T = a.tokens();
    std::vector<long long> assigned(n, 0);
    long long ndrop = 0;
    if (T > 0) {
        DeviceAssignment d(a);
        DevBuf<int64_t> load(n), asg(n), nd(1);
        check(moe_balance_counts(d.experts.p, d.dropped.p, T, a.num_experts, a.top_k, n, load.p,
                                 asg.p, nd.p, nullptr));
        const auto l = load.download(n), g = asg.download(n);
        s.per_group_load.assign(l.begin(), l.end());
        assigned.assign(g.begin(), g.end());
        ndrop = nd.download(1)[0];
    }
    const long long tl = std::accumulate(s.per_group_load.begin(), s.per_group_load.end(), 0ll);
    const long long ta = std::accumulate(assigned.begin(), assigned.end(), 0ll);
    double loss = 0.0;
    if (tl > 0 && ta > 0) {
        for (long long g = 0; g < n; ++g)
            loss += (double(s.per_group_load[g]) / double(tl)) * (double(assigned[g]) / double(ta));
        loss *= double(n);
    }
    s.balance_loss_value = loss;
    s.capacity = T > 0 ? (long long)std::ceil(double(T) * double(a.top_k) / double(n)) : 0;
    s.drop_rate = T > 0 ? double(ndrop) / double(T) : 0.0;
    return s;
}

// Versioned JSON (schema_version 1, docs/schemas.md:98-129).
nlohmann::json to_json(const RoutingAssignment& a) {
    nlohmann::json j;
    j["schema_version"] = 1;
    j["num_experts"] = a.num_experts;
    j["top_k"] = a.top_k;
    j["n_groups"] = a.n_groups;
    j["experts"] = a.experts;
    j["source_rank"] = a.source_rank;
    j["dropped"] = std::vector<int>(a.dropped.begin(), a.dropped.end());
    return j;
}

nlohmann::json to_json(const TileLayout& t) {
    nlohmann::json j;
    j["schema_version"] = 1;
    j["tile_rows"] = t.tile_rows;
    j["tiles"] = nlohmann::json::array();
    for (const Tile& tile : t.tiles)
        j["tiles"].push_back({{"expert", tile.expert}, {"row_begin", tile.row_begin},
                              {"row_end", tile.row_end}, {"dependent_ranks", tile.dependent_ranks}});
    return j;
}

RoutingAssignment assignment_from_json(const nlohmann::json& j) {
    if (j.at("schema_version").get<int>() != 1)
        throw std::runtime_error("unsupported routing schema version");
    RoutingAssignment a;
    a.num_experts = j.at("num_experts").get<long long>();
    a.top_k = j.at("top_k").get<long long>();
    a.n_groups = j.at("n_groups").get<long long>();
    a.experts = j.at("experts").get<std::vector<std::vector<int>>>();
    a.source_rank = j.at("source_rank").get<std::vector<int>>();
    const auto d = j.at("dropped").get<std::vector<int>>();
    a.dropped.assign(d.begin(), d.end());
    return a;
}

}  // namespace moeplan::routing
