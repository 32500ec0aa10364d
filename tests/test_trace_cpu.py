"""CPU checks of the measured-timeline tooling: %globaltimer stamp summaries
(rank alignment on the first barrier's release, barrier waits separated from
busy time) and the reference-schema trace writer."""
import copy
import json
import os

from paper_2505_11432_b200.trace import stamp_summary, write_stamp_trace

PH = ["route", "permute", "dispatch", "fc1", "fc2", "combine", "fwd_end", "dispatch_dy", "fc2_dgrad",
      "fc1_dgrad", "dgate", "combine_dx", "fc2_wgrad", "fc1_wgrad", "router_wgrad", "end"]


def _rank(rank, offset_ns, fc1_us, wait1_us):
    t = offset_ns
    phases, bars = {}, {}
    dur = {"route": 50, "permute": 50, "dispatch": 10, "fc1": fc1_us, "fc2": 700 + wait1_us, "combine": 20,
           "fwd_end": 1, "dispatch_dy": 30, "fc2_dgrad": 800, "fc1_dgrad": 1400, "dgate": 20, "combine_dx": 20,
           "fc2_wgrad": 600, "fc1_wgrad": 1300, "router_wgrad": 30, "end": 0}
    for p in PH:
        phases[p] = t
        if p == "route":
            bars["0"] = (t + 10_000, t + 40_000)          # metadata barrier: released at +40 us
        if p == "fc2":
            bars["1"] = (t + 700_000, t + (700 + wait1_us) * 1000)
        t += dur[p] * 1000
    return {"rank": rank, "steps": [{"phases": phases, "barriers": bars}]}


def test_stamp_summary_aligns_ranks_and_separates_barrier_waits(tmp_path):
    # rank 1's clock is 5 ms ahead; its fc1 is 100 us slower, so rank 0 waits 100 us at barrier 1
    r0 = _rank(0, 0, 1300, 100)
    r1 = _rank(1, 5_000_000, 1400, 0)
    s = stamp_summary([r0, r1])["summary"]
    assert abs(s["makespan_ms"]["median"] - (sum([50, 50, 10, 1400, 700, 20, 30, 800, 1400, 20, 20, 600, 1300, 30])
                                             + 1) / 1000) < 0.2, s["makespan_ms"]
    assert abs(s["barrier_wait_ms"]["slot1_fc2"] - 0.1) < 1e-6
    assert abs(s["phases_busy_ms"]["fc2"] - 0.7) < 1e-6      # the wait is not busy time
    assert s["per_rank_busy_gemm_ms"]["1"]["fc1"] == 1.4
    out = tmp_path / "t.json"
    write_stamp_trace(str(out), stamp_summary([r0, r1]), 8192, 4096, 14336, 0.0)
    d = json.loads(out.read_text())
    assert d["schema_version"] == 1
    x = [e for e in d["traceEvents"] if e["ph"] == "X"]
    assert {e["pid"] for e in x} == {0, 1}
    # aligned: both ranks' route events start at ts 0 (same physical time)
    starts = {e["pid"]: e["ts"] for e in x if e["name"] == "route"}
    assert abs(starts[0] - starts[1]) < 1e-6, starts


def test_reference_cost_model_driver():
    """oracle/_ref/ref_model (the reference's graph/schedule/commcost compiled
    unmodified) prints the modelled layer timeline; its fused pairs are never
    slower than the unfused operators (schedule.cpp:379), and the FFN nodes
    the measured-vs-modelled diff groups are all present."""
    import subprocess
    import pytest
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "oracle", "_ref", "ref_model")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_model not built (needs /root/reference)")
    for pattern in ("a2a", "ag_rs"):
        out = subprocess.run([exe, "4096", "14336", "8", "2", "4096", "4", pattern, "bf16", "1684.4e12",
                              "6535.1e9", "900e9"], capture_output=True, text=True, check=True).stdout
        d = json.loads(out)
        for ph in ("forward", "backward"):
            for p in d[ph]["fused_pairs"]:
                assert p["fused_us"] <= p["unfused_us"] + 1e-6, p
        names = {e["name"] for e in d["forward"]["unfused"]["events"]}
        assert {"router", "fc1", "swiglu", "weighted_sum", "fc2"} <= names
        assert ("a2a_dispatch" in names) == (pattern == "a2a") and ("ag_ffn_in" in names) == (pattern == "ag_rs")
