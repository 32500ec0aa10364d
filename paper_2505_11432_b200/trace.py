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
