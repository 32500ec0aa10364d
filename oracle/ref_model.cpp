// ref_model.cpp — drives the REFERENCE's own cost model / scheduler
// (/root/reference/proj/core/src/{graph,schedule,commcost,...}.cpp, compiled
// unmodified from where they lie by oracle/Makefile into oracle/_ref/) for
// one MoE layer at the B200 parameters, and prints the modelled per-operator
// timeline as JSON so bench / profile measurements can be diffed against it
// (SURVEY §8f row 2; schedule.cpp:88-154 inter-op schedule, :205-380 fused
// pairs, trace.cpp:44-78 trace events).
//
// TEST / MEASUREMENT INFRASTRUCTURE ONLY (scripts/model_vs_measured.py).
//
// usage: ref_model h f E k tokens_per_rank n ep_pattern(a2a|ag_rs) comm(bf16|fp8_e4m3)
//                  peak_flops mem_bw intra_bw
#include <cstdio>
#include <cstdlib>
#include <string>

#include <nlohmann/json.hpp>

#include "moeplan/config.hpp"
#include "moeplan/memmodel.hpp"
#include "moeplan/simsched.hpp"

using namespace moeplan;
using namespace moeplan::simsched;

static nlohmann::json timeline_json(const OpGraph& g, const Timeline& t) {
    nlohmann::json ev = nlohmann::json::array();
    for (const auto& e : t.events) {
        const auto& node = g.at(e.node);
        ev.push_back({{"name", e.name},
                      {"kind", op_kind_name(node.kind)},
                      {"start_us", e.start * 1e6},
                      {"dur_us", (e.end - e.start) * 1e6},
                      {"lane", e.resource == StreamClass::compute      ? "compute"
                               : e.resource == StreamClass::comm_intra ? "comm_intra"
                                                                       : "comm_inter"},
                      {"flops", node.flops},
                      {"bytes", node.kind == OpKind::collective ? (double)node.volume.bytes : node.bytes_moved}});
    }
    return {{"events", ev},
            {"makespan_us", t.makespan * 1e6},
            {"busy_compute_us", t.busy_compute * 1e6},
            {"exposed_comm_us", t.exposed_comm * 1e6}};
}

int main(int argc, char** argv) {
    if (argc < 12) {
        std::fprintf(stderr, "usage: %s h f E k tokens_per_rank n ep_pattern comm peak mem_bw intra_bw\n", argv[0]);
        return 2;
    }
    try {
        ModelConfig model;
        model.name = "moe_layer";
        model.hidden_size = std::atoll(argv[1]);
        model.ffn_hidden_size = std::atoll(argv[2]);
        model.num_experts = std::atoll(argv[3]);
        model.top_k = std::atoll(argv[4]);
        const long long tr = std::atoll(argv[5]);
        const long long n = std::atoll(argv[6]);
        model.micro_batch = 1;
        model.seq_len = tr * n;  // b*s/n rows per rank = tokens per rank
        model.num_heads = 64;
        model.query_kv_ratio = 8;
        model.vocab_size = 32000;
        model.num_layers = 1;
        model.global_batch = 1;
        ParallelismPlan plan;
        plan.n = n;
        plan.ep_pattern = std::string(argv[7]) == "ag_rs" ? commcost::EpPattern::ag_rs : commcost::EpPattern::a2a;
        PrecisionConfig prec;
        if (std::string(argv[8]) == "fp8_e4m3") {
            prec.tp_comm_format = Format::fp8_e4m3;
            prec.quant_granularity = "per_token";
        }
        ClusterConfig cl;
        cl.name = "b200";
        cl.gpus_per_node = 8;
        cl.peak_flops = std::atof(argv[9]);
        cl.mem_bw = std::atof(argv[10]);
        cl.intra_bw = std::atof(argv[11]);
        cl.sm_count = 148;
        cl.mem_capacity = 180e9;
        const EfficiencyTable eff;
        const auto link = commcost::LinkModel::from_cluster(cl);

        nlohmann::json out;
        for (int bwd = 0; bwd < 2; ++bwd) {
            OpGraph g = bwd ? build_backward_graph(plan, model, prec, memmodel::RematPolicy::selective())
                            : build_layer_graph(plan, model, prec);
            cost_graph(g, cl, eff, link);
            const Timeline unfused = schedule(g, ScheduleMode::inter_op);
            nlohmann::json pairs = nlohmann::json::array();
            auto fus = default_fusions(g);
            for (const auto& p : fus)
                pairs.push_back({{"comm", g.at(p.comm_node).name},
                                 {"compute", g.at(p.compute_node).name},
                                 {"unfused_us", (g.at(p.comm_node).cost + g.at(p.compute_node).cost) * 1e6},
                                 {"fused_us", fused_overlap_time(g, p, cl) * 1e6}});
            const OpGraph fg = apply_intra_op(g, select_fusions(g, cl), cl);
            const Timeline fused = schedule(fg, ScheduleMode::inter_op);
            out[bwd ? "backward" : "forward"] = {{"unfused", timeline_json(g, unfused)},
                                                 {"fused", timeline_json(fg, fused)},
                                                 {"fused_pairs", pairs}};
        }
        out["params"] = {{"h", model.hidden_size}, {"f", model.ffn_hidden_size}, {"E", model.num_experts},
                         {"k", model.top_k}, {"tokens_per_rank", tr}, {"n", n}, {"ep_pattern", argv[7]},
                         {"comm", argv[8]}, {"peak_flops", cl.peak_flops}, {"mem_bw", cl.mem_bw},
                         {"intra_bw", cl.intra_bw},
                         {"efficiency", {{"gemm", eff.gemm}, {"grouped_gemm", eff.grouped_gemm},
                                         {"memory_bound", eff.memory_bound}}}};
        std::printf("%s\n", out.dump().c_str());
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_model: %s\n", e.what());
        return 1;
    }
}
