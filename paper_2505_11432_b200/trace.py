"""Measured layer timeline in the reference's trace-event schema
(docs/schemas.md:74-96, trace.cpp:44-78): one complete event per operator
phase, lanes compute / comm_intra / comm_inter, so measured and modelled
(`moeplan simulate --trace`) timelines can be diffed.

Phases are CUDA-event intervals on the layer stream (sequential); the fused
AG-GEMM / GEMM-RS kernels carry their communication inside the compute lane.
"""
from __future__ import annotations

import json

KINDS = {
    "route": "router", "permute": "scatter", "dispatch": "scatter", "fc1": "fused", "fc2": "fused",
    "combine": "gather", "dispatch_dy": "scatter", "fc2_dgrad": "fused", "fc1_dgrad": "fused",
    "dgate": "weighted_sum", "combine_dx": "gather", "fc2_wgrad": "grouped_gemm",
    "fc1_wgrad": "grouped_gemm", "router_wgrad": "router",
}


def phase_flops(name: str, rows: int, h: int, f: int) -> float:
    return {"fc1": 2.0 * rows * h * 2 * f, "fc2": 2.0 * rows * f * h,
            "fc2_dgrad": 2.0 * rows * h * f, "fc1_dgrad": 2.0 * rows * 2 * f * h,
            "fc2_wgrad": 2.0 * rows * h * f, "fc1_wgrad": 2.0 * rows * 2 * f * h}.get(name, 0.0)


def trace_events(phases_ms: dict, rows: int, h: int, f: int, exposed_comm_s: float | None = None) -> dict:
    events = [{"ph": "M", "pid": 0, "tid": tid, "name": "thread_name", "args": {"name": lane}}
              for tid, lane in enumerate(("compute", "comm_intra", "comm_inter"))]
    ts = 0.0
    for name, ms in phases_ms.items():
        dur_us = ms * 1000.0
        events.append({"ph": "X", "pid": 0, "tid": 0, "name": name, "ts": ts, "dur": dur_us,
                       "args": {"kind": KINDS.get(name, "fused"), "flops": phase_flops(name, rows, h, f),
                                "bytes": 0.0, "remat": name == "fc2_dgrad"}})
        ts += dur_us
    return {"schema_version": 1, "displayTimeUnit": "ns", "traceEvents": events,
            "makespan_seconds": ts * 1e-6,
            "exposed_comm_seconds": 0.0 if exposed_comm_s is None else max(exposed_comm_s, 0.0)}


def write_trace(path: str, phases_ms: dict, rows: int, h: int, f: int, exposed_comm_s=None) -> None:
    with open(path, "w") as fh:
        json.dump(trace_events(phases_ms, rows, h, f, exposed_comm_s), fh, indent=1)


PHASE_ORDER = ("route", "permute", "dispatch", "fc1", "fc2", "combine", "fwd_end", "dispatch_dy", "fc2_dgrad",
               "fc1_dgrad", "dgate", "combine_dx", "fc2_wgrad", "fc1_wgrad", "router_wgrad", "end")
# the phase whose interval contains each barrier slot's wait (layer.cu)
BARRIER_PHASE = {0: "route", 1: "fc2", 2: "dispatch_dy", 3: "dgate"}


def _intervals(phases_ns: dict):
    names = [p for p in PHASE_ORDER if p in phases_ns]
    out = []
    for a, b in zip(names, names[1:]):
        if a == "fwd_end":
            continue
        out.append((a, phases_ns[a], phases_ns[b]))
    return out


def stamp_summary(all_ranks: list) -> dict:
    """%globaltimer stamps of graph-replayed steps from every rank ->
    per-phase durations (median over steps of the max over ranks), step
    makespan, and the flag-barrier waits (time a rank idles for the slowest
    one: rank imbalance / skew, not link time — the fused kernels carry the
    NVLink traffic inside the compute phases)."""
    import numpy as np
    nsteps = min(len(r["steps"]) for r in all_ranks)
    per_phase, busy_phase, makespans, waits = {}, {}, [], {}
    for s in range(nsteps):
        starts, ends = [], []
        dur, busy = {}, {}
        for r in all_ranks:
            st = r["steps"][s]
            iv = _intervals(st["phases"])
            if not iv:
                continue
            # the GPUs' %globaltimer clocks are not aligned: put every rank on
            # rank 0's clock through the first barrier's release, which all
            # ranks leave at the same physical time (to within the flag latency)
            off = 0
            b0 = st["barriers"].get("0") or st["barriers"].get(0)
            r0 = all_ranks[0]["steps"][s]["barriers"]
            b0_ref = r0.get("0") or r0.get(0)
            if b0 and b0_ref:
                off = b0_ref[1] - b0[1]
            starts.append(iv[0][1] + off)
            ends.append(iv[-1][2] + off)
            wait_in = {}
            for slot, (e0, e1) in st["barriers"].items():
                waits.setdefault(int(slot), []).append((s, (e1 - e0) / 1e6))
                wait_in[BARRIER_PHASE[int(slot)]] = (e1 - e0) / 1e6
            for name, a, b in iv:
                dur.setdefault(name, []).append((b - a) / 1e6)
                busy.setdefault(name, []).append((b - a) / 1e6 - wait_in.get(name, 0.0))
        if starts:
            makespans.append((max(ends) - min(starts)) / 1e6)
        for name, v in dur.items():
            per_phase.setdefault(name, []).append(max(v))
        for name, v in busy.items():
            busy_phase.setdefault(name, []).append(max(v))
    # per-rank busy time of the GEMM phases (median over steps): separates a
    # slower GPU (clock / power) from routing imbalance
    per_rank = {}
    for r in all_ranks:
        acc = {}
        for s_ in range(nsteps):
            st = r["steps"][s_]
            wait_in = {BARRIER_PHASE[int(k_)]: (v_[1] - v_[0]) / 1e6 for k_, v_ in st["barriers"].items()}
            for name, a, b in _intervals(st["phases"]):
                acc.setdefault(name, []).append((b - a) / 1e6 - wait_in.get(name, 0.0))
        per_rank[str(r["rank"])] = {k_: round(float(np.median(v_)), 4) for k_, v_ in acc.items()
                                    if k_ in ("fc1", "fc2", "fc2_dgrad", "fc1_dgrad", "fc2_wgrad", "fc1_wgrad")}
    wait_med = {}
    for slot, lst in waits.items():
        by_step = {}
        for s, w in lst:
            by_step[s] = max(by_step.get(s, 0.0), w)
        wait_med[slot] = float(np.median(list(by_step.values())))
    summary = {
        "steps": nsteps, "ranks": len(all_ranks),
        "makespan_ms": {"median": float(np.median(makespans)), "min": float(np.min(makespans)),
                        "max": float(np.max(makespans))} if makespans else None,
        "phases_ms": {k: round(float(np.median(v)), 4) for k, v in per_phase.items()},
        "phases_busy_ms": {k: round(float(np.median(v)), 4) for k, v in busy_phase.items()},
        "barrier_wait_ms": {f"slot{k}_{BARRIER_PHASE[k]}": round(v, 4) for k, v in sorted(wait_med.items())},
        "rank_imbalance_idle_ms": round(sum(wait_med.values()), 4),
        "per_rank_busy_gemm_ms": per_rank,
        "how": "device %globaltimer stamps at each phase boundary and at every flag barrier's entry/release, "
               "inside graph-replayed steps (each replay synchronised and read back); ranks aligned on the first "
               "barrier's release; phase = median over steps of the max over ranks; phases_busy = the same minus "
               "the barrier wait inside the phase; barrier wait = time a rank idles at the barrier for the "
               "slowest rank (rank imbalance / skew)",
    }
    return {"summary": summary, "raw": all_ranks}


def write_stamp_trace(path: str, gtrace: dict, rows: int, h: int, f: int, exposed_comm_s=None) -> None:
    """Trace-event file (reference schema, trace.cpp:44-78) of the LAST
    graph-replayed step: one process per rank on the shared device clock,
    phases on the compute lane, barrier waits on comm_intra."""
    raw = gtrace["raw"]
    step = min(len(r["steps"]) for r in raw) - 1

    def offset(r):
        b = r["steps"][step]["barriers"]
        b0 = b.get("0") or b.get(0)
        r0 = raw[0]["steps"][step]["barriers"]
        ref = r0.get("0") or r0.get(0)
        return (ref[1] - b0[1]) if (b0 and ref) else 0

    t0 = min(min(r["steps"][step]["phases"].values()) + offset(r) for r in raw)
    events = []
    for r in raw:
        pid = r["rank"]
        t0r = t0 - offset(r)
        for tid, lane in enumerate(("compute", "comm_intra", "comm_inter")):
            events.append({"ph": "M", "pid": pid, "tid": tid, "name": "thread_name", "args": {"name": lane}})
        st = r["steps"][step]
        for name, a, b in _intervals(st["phases"]):
            events.append({"ph": "X", "pid": pid, "tid": 0, "name": name, "ts": (a - t0r) / 1e3,
                           "dur": (b - a) / 1e3,
                           "args": {"kind": KINDS.get(name, "fused"), "flops": phase_flops(name, rows, h, f),
                                    "bytes": 0.0, "remat": name == "fc2_dgrad"}})
        for slot, (e0, e1) in st["barriers"].items():
            events.append({"ph": "X", "pid": pid, "tid": 1, "name": f"barrier_wait_{BARRIER_PHASE[int(slot)]}",
                           "ts": (e0 - t0r) / 1e3, "dur": (e1 - e0) / 1e3,
                           "args": {"kind": "idle", "flops": 0.0, "bytes": 0.0, "remat": False}})
    summ = gtrace["summary"]
    out = {"schema_version": 1, "displayTimeUnit": "ns", "traceEvents": events,
           "makespan_seconds": (summ["makespan_ms"]["median"] / 1e3) if summ["makespan_ms"] else 0.0,
           "exposed_comm_seconds": exposed_comm_s,
           "rank_imbalance_idle_seconds": summ["rank_imbalance_idle_ms"] / 1e3,
           "summary": summ}
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
