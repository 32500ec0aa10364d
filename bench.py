#!/usr/bin/env python
"""Benchmark: MoE layer forward+backward tokens/s on B200 (BASELINE.json
metric), Mixtral-8x7B-shape layer (configs[1]): hidden 4096, ffn 14336,
8 experts top-2, bf16, 4096 tokens per rank, EP = number of GPUs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0. Under torchrun (N > 1) every rank runs one process
per GPU; the layer's dispatch/combine go over NVLink inside the kernels.

`--impl reference`: the reference's CPU path on this host (rank 0 only):
its own routing code (oracle/_ref, compiled from the reference sources) plus
the fp32 oracle port of the dense math (the reference has none), on a bounded
token sample per step.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "mixtral": dict(workload="mixtral-8x7b-moe-layer-fwd+bwd", hidden=4096, ffn_hidden=14336,
                    num_experts=8, top_k=2, tokens_per_rank=4096),
    "deepseek": dict(workload="deepseek-v3-moe-layer-fwd+bwd", hidden=7168, ffn_hidden=2048,
                     num_experts=256, top_k=8, tokens_per_rank=4096),
    "small": dict(workload="small-moe-layer-fwd+bwd", hidden=1024, ffn_hidden=2816,
                  num_experts=8, top_k=2, tokens_per_rank=4096),
    # configs[0] as BASELINE states it: fp32 forward on one GPU (FFMA grouped GEMMs)
    "small_f32": dict(workload="small-moe-layer-fwd-fp32", hidden=1024, ffn_hidden=2816,
                      num_experts=8, top_k=2, tokens_per_rank=4096),
    # configs[4]: Mixtral shape, FP8 dispatch/combine, gate after fc2,
    # Zipf(1.2) routing from the reference's own simulate_routing (golden fixture)
    "mixtral_fp8_zipf": dict(workload="mixtral-8x7b-moe-layer-fwd+bwd-fp8comm-zipf1.2", hidden=4096,
                             ffn_hidden=14336, num_experts=8, top_k=2, tokens_per_rank=4096,
                             comm="fp8", gate="after_fc2_out",
                             routing_fixture="tests/golden/routing_cfg5_zipf_nodrop_n8.npz"),
    # FP8 communication with the learned router (uniform-ish load): the cost of the
    # E4M3 quantise / dequantise against the halved NVLink bytes
    "mixtral_fp8": dict(workload="mixtral-8x7b-moe-layer-fwd+bwd-fp8comm", hidden=4096, ffn_hidden=14336,
                        num_experts=8, top_k=2, tokens_per_rank=4096, comm="fp8", gate="after_fc2_out"),
    # configs[3]: sequence-parallel attention QKV / out-proj, hidden 8192, seq 8192, GQA m=8
    "attn": dict(workload="sp-attention-qkv-ag-gemm+out-proj-gemm-rs", hidden=8192, seq=8192, gqa=8),
    # §8f row 3: Ulysses SP projections (the paper's attention strategy) at the
    # same cfg4 geometry
    "ulysses": dict(workload="ulysses-sp-attention-qkv-gemm-a2a+a2a-out-proj-gemm", hidden=8192, seq=8192, gqa=8),
    # §8f row 4: DP gradient sync with bf16 compression; gradient = one
    # Mixtral expert's W1 + W2 (3 * 4096 * 14336 fp32), the per-rank expert
    # parameters at EP = 8
    "dp": dict(workload="dp-grad-sync-bf16-a2a-fp32-reduce", count=3 * 4096 * 14336),
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sus=d["bf16_tflops_sustained"],
                    src="measured")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region via NVML
    (every ~20 ms; falls back to nvidia-smi polling if NVML is unavailable)."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []  # (sm_mhz, max_mhz, reason_bits)
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        import pynvml as N
        N.nvmlInit()
        hd = N.nvmlDeviceGetHandleByIndex(self.idx)
        mx = N.nvmlDeviceGetMaxClockInfo(hd, N.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                self.samples.append((N.nvmlDeviceGetClockInfo(hd, N.NVML_CLOCK_SM), mx,
                                     N.nvmlDeviceGetCurrentClocksEventReasons(hd)))
            except Exception:
                pass
            self._stop.wait(0.02)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        bits = (0x8, 0x40, 0x20, 0x4)
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip().split(",")
                rb = sum(b for b, v in zip(bits, out[2:]) if v.strip() == "Active")
                self.samples.append((float(out[0]), float(out[1]), rb))
            except Exception:
                pass
            self._stop.wait(0.2)

    def start(self):
        try:
            import pynvml  # noqa: F401
            target = self._run_nvml
        except Exception:
            target = self._run_smi
        self._t = threading.Thread(target=target, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for s in self.samples for name, bit in self.REASONS if s[2] & bit})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(s[1] for s in self.samples) if self.samples else None,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml"}


class NvlinkCounters:
    """Cumulative NVLink data bytes of one GPU from NVML field values
    (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX, KiB, summed over links):
    read before and after a timed region, they give the bytes the fused
    kernels actually put on the links (payload, no protocol overhead)."""

    TX, RX = 138, 139

    def __init__(self, gpu_index: int):
        import pynvml as N
        N.nvmlInit()
        self.N = N
        self.hd = N.nvmlDeviceGetHandleByIndex(gpu_index)
        self.links = []
        for link in range(18):
            try:
                if N.nvmlDeviceGetNvLinkState(self.hd, link) == N.NVML_FEATURE_ENABLED:
                    self.links.append(link)
            except Exception:
                pass

    def probe(self):
        """True when the driver exposes the counters (NOT_SUPPORTED on some pools)."""
        N = self.N
        for link in self.links[:1]:
            v = N.nvmlDeviceGetFieldValues(self.hd, [(self.TX, link)])[0]
            return v.nvmlReturn == 0
        return False

    def read(self):
        N = self.N
        tx = rx = 0
        for link in self.links:
            vals = N.nvmlDeviceGetFieldValues(self.hd, [(self.TX, link), (self.RX, link)])
            for v, acc in zip(vals, ("tx", "rx")):
                if v.nvmlReturn != 0:
                    continue
                x = getattr(v.value, "ullVal", 0) or getattr(v.value, "ulVal", 0)
                if acc == "tx":
                    tx += x
                else:
                    rx += x
        return tx * 1024, rx * 1024


_CPU_STATE = {}


def _cpu_weights(E, f, h):
    """fp32 expert + router weights for the CPU baseline (generated once, not
    timed). Values only set the timing, so a 64 MB N(0,1) block is tiled."""
    key = (E, f, h)
    if key not in _CPU_STATE:
        _CPU_STATE.clear()
        rng = np.random.default_rng(0)
        blk = rng.standard_normal(1 << 24, dtype=np.float32)

        def fill(shape, scale):
            a = np.empty(shape, np.float32)
            flat = a.reshape(-1)
            for o in range(0, flat.size, blk.size):
                m = min(blk.size, flat.size - o)
                np.multiply(blk[:m], np.float32(scale), out=flat[o:o + m])
            return a
        w1 = fill((E, 2 * f, h), h ** -0.5)
        w2 = fill((E, h, f), f ** -0.5)
        wr = fill((E, h), h ** -0.5)
        grads = (np.empty_like(w1), np.empty_like(w2), np.empty((E, h), np.float32))
        _CPU_STATE[key] = (w1, w2, wr, grads)
    return _CPU_STATE[key]


def cpu_reference_step(cfg, n_ranks, max_dense_tokens=4096, seed=0):
    """One step of the reference CPU path for the whole job (T = n_ranks x T_r
    tokens): the reference's own routing code (oracle/_ref, single-threaded as
    shipped: build_scatter_map + sort_tokens_for_tiles for every rank,
    balance_metrics) on all T tokens, and the dense layer (router, fc1, SwiGLU,
    fc2, combine, full backward incl. weight gradients) as fp32 numpy/OpenBLAS
    on all host cores for min(T, max_dense_tokens) tokens. Returns a dict; the
    step time is t_route + t_dense * T / S (S = T at N = 1: no extrapolation)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as P
    from threadpoolctl import threadpool_limits
    h, f, E, k, Tr = cfg["hidden"], cfg["ffn_hidden"], cfg["num_experts"], cfg["top_k"], cfg["tokens_per_rank"]
    T = n_ranks * Tr
    S = min(T, max_dense_tokens)
    w1, w2, wr, grads = _cpu_weights(E, f, h)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((S, h), dtype=np.float32) * np.float32(0.5)
    dy = rng.standard_normal((S, h), dtype=np.float32) * np.float32(0.1)
    cores = os.cpu_count() or 1
    kind = "reference" if P.ref_available() else "port"
    # routing input for all T tokens (simulate_routing = the reference's input generator, not timed)
    if kind == "reference":
        ex, src, dr = P.ref_simulate_routing(T, E, k, "random", 11 + seed, n_groups=n_ranks)
        t_route = float(np.sum(P.ref_time_routing(ex, src, dr, E, n_ranks, 128, 1))) / 1000.0
    else:
        ex = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
        src = (np.arange(T) // Tr).astype(np.int32)
        dr = np.zeros(T, np.uint8)
        t0 = time.perf_counter()
        for r in range(n_ranks):
            P.orc_build_scatter_map(ex, src, dr, E, n_ranks, r)
        t_route = time.perf_counter() - t0
    with threadpool_limits(limits=cores):
        t0 = time.perf_counter()
        P.np_moe_fwd_bwd(x, dy, wr, w1, w2, k, out=grads)
        t_dense = time.perf_counter() - t0
    t_step = t_route + t_dense * T / S
    return dict(t_step=t_step, t_route=t_route, t_dense=t_dense, T=T, S=S, kind=kind, cores=cores,
                value=T / t_step)


def _cpu_sample_text(r):
    ext = "" if r["S"] == r["T"] else f", dense time scaled x{r['T'] / r['S']:.0f} from {r['S']} tokens"
    return (f"whole job per step: {r['T']} tokens; reference routing maps for every rank + tile layout + "
            f"balance (oracle/_ref, 1 thread, {1000 * r['t_route']:.1f} ms) + fp32 numpy/OpenBLAS dense "
            f"router+FFN fwd+bwd incl. weight grads on {r['cores']} threads ({r['t_dense']:.2f} s{ext})")


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.gpus
    times = []
    last = None
    for i in range(args.warmup + args.steps):
        # warm-up steps run the same code on a small dense sample (pages, BLAS threads)
        r = cpu_reference_step(cfg, n, max_dense_tokens=(256 if i < args.warmup else 4096), seed=i)
        if i >= args.warmup:
            times.append(r["t_step"])
            last = r
    ms = 1000.0 * float(np.mean(times))
    val = n * cfg["tokens_per_rank"] / (ms / 1000.0)
    line = {
        "impl": "reference", "metric": "moe_layer_fwd_bwd_tokens_per_s", "value": val,
        "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["workload"], "hidden": cfg["hidden"], "ffn_hidden": cfg["ffn_hidden"],
                   "num_experts": cfg["num_experts"], "top_k": cfg["top_k"],
                   "tokens_per_rank": cfg["tokens_per_rank"], "global_tokens": n * cfg["tokens_per_rank"],
                   "dense_tokens_per_step": last["S"]},
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": last["cores"], "kind": last["kind"],
                         "sample": _cpu_sample_text(last)},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def layer_pad(L) -> int:
    # expert segments are padded to 128 rows (layer.cu; CTA pairs run a segment's
    # odd 128-row block as an M = 128 pair tile)
    return 128


def routing_probe_rows(L, rank, el):
    cnt = L.routing()["per_expert_counts"].cpu().tolist()[rank * el:(rank + 1) * el]
    p = layer_pad(L)
    return int(sum((c + p - 1) // p * p for c in cnt))


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2505_11432_b200 import launch_count, launch_count_reset
    from paper_2505_11432_b200.layer import MoELayer

    h, f, E, k, Tr = cfg["hidden"], cfg["ffn_hidden"], cfg["num_experts"], cfg["top_k"], cfg["tokens_per_rank"]
    n = world
    el = E // n
    g = torch.Generator(device="cuda").manual_seed(42)
    w1 = (torch.randn(el, 2 * f, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
    w2 = (torch.randn(el, h, f, device="cuda", generator=g) / f ** 0.5).bfloat16()
    wr = (torch.randn(E, h, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7)) / h ** 0.5).bfloat16()
    injected = "routing_fixture" in cfg
    L = MoELayer(Tr, h, f, E, k, ep_size=n, rank=rank, capacity_factor=0.0,
                 gate_order=cfg.get("gate", "before_fc2_in"), comm_format=cfg.get("comm", "bf16"),
                 route_mode="injected" if injected else "learned", ep_pattern=args.ep_pattern,
                 remat=not args.no_remat)
    L.set_weights(w1, w2, wr)
    if injected:
        # routing input data: the reference's simulate_routing output (committed fixture)
        fx = np.load(os.path.join(ROOT, cfg["routing_fixture"]))
        ex_all = fx["experts"].astype(np.int32).reshape(-1, k)
        assert ex_all.shape[0] >= Tr * n, "fixture too small for this many ranks"
        ex_loc = ex_all[rank * Tr:(rank + 1) * Tr]
        glog = np.random.default_rng(rank).standard_normal((Tr, k)).astype(np.float32)
        gates = np.exp(glog) / np.exp(glog).sum(1, keepdims=True)
        L.set_routing(torch.from_numpy(np.ascontiguousarray(ex_loc)).cuda(), torch.from_numpy(gates).cuda())
    del w1, w2
    if n > 1:
        L.connect()
    gx = torch.Generator(device="cuda").manual_seed(1234 + rank)
    x = (torch.randn(Tr, h, device="cuda", generator=gx) * 0.5).bfloat16()
    dy = (torch.randn(Tr, h, device="cuda", generator=gx) * 0.1).bfloat16()
    L.input_buffer.copy_(x)
    L.dy_buffer.copy_(dy)          # inputs resident in the layer's own (symmetric) buffers
    dy = L.dy_buffer
    dx = torch.empty(Tr, h, dtype=torch.bfloat16, device="cuda")
    dw1 = torch.empty(el, 2 * f, h, dtype=torch.bfloat16, device="cuda")
    dw2 = torch.empty(el, h, f, dtype=torch.bfloat16, device="cuda")
    dwr = torch.empty(E, h, dtype=torch.float32, device="cuda")
    y = torch.empty(Tr, h, dtype=torch.bfloat16, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        L.forward(None, y)
        L.backward(dy, dx, dw1, dw2, dwr)

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    sync_all()
    if L.error_flag():
        raise RuntimeError("cross-GPU flag wait timed out during warm-up")
    run_step = step
    launch_count_reset()
    step()
    per_step_launches = launch_count()
    sync_all()
    if not args.no_graph:
        # the whole fwd+bwd step (router, maps, GEMMs, NVLink barriers) as one CUDA graph
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        sync_all()
        run_step = graph.replay

    # ---- device-timed region (inputs resident in HBM) ----
    nvl = None
    if world > 1:
        try:
            nvl = NvlinkCounters(local)
            if not nvl.probe():
                nvl = None
        except Exception:  # noqa: BLE001
            nvl = None
    nvl0 = nvl.read() if nvl else None
    clocks = ClockSampler(local)
    clocks.start()
    launch_count_reset()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sync_all()
    ev0.record(stream)
    for _ in range(args.steps):
        run_step()
    ev1.record(stream)
    sync_all()
    launches = launch_count() if args.no_graph else per_step_launches * args.steps
    clk = clocks.stop()
    nvl_meas = None
    if nvl:
        tx1, rx1 = nvl.read()
        nvl_meas = [(tx1 - nvl0[0]) / args.steps, (rx1 - nvl0[1]) / args.steps]
    ms_local = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms_local], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = n * Tr / (ms / 1000.0)

    # ---- exposed communication: T_layer - T_compute_only (schedule.cpp:149-152) ----
    exposed = None
    if world > 1:
        # exposed = T_layer - T_compute_only (schedule.cpp:149-152). Both modes run
        # as captured CUDA graphs of the same kernels (compute-only: peer buffers
        # replaced by local ones, no barriers); 10 alternating windows so clock
        # drift shows up as spread instead of masquerading as communication.
        def capture(compute_only):
            L.set_compute_only(compute_only)
            for _ in range(2):
                step()
            sync_all()
            if args.no_graph:
                return step
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                step()
            gr.replay()
            sync_all()
            return gr.replay
        run_co = capture(True)
        run_norm = capture(False)
        wsteps = max(5, args.steps // 2)

        def window(fn):
            sync_all()
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            for _ in range(wsteps):
                fn()
            c1.record(stream)
            sync_all()
            tc = torch.tensor([c0.elapsed_time(c1) / wsteps], device="cuda")
            dist.all_reduce(tc, op=dist.ReduceOp.MAX)
            return float(tc.item())
        t_norm, t_comp = [], []
        for _ in range(10):
            t_norm.append(window(run_norm))
            t_comp.append(window(run_co))
        # per-phase times in compute-only mode (where the step goes without NVLink)
        L.set_compute_only(True)
        L.enable_timing(True)
        L.forward(None, y)
        L.backward(dy, dx, dw1, dw2, dwr)
        phases_co = L.phase_times()
        L.enable_timing(False)
        L.set_compute_only(False)
        for _ in range(2):
            step()
        sync_all()
        tn, tcm = float(np.median(t_norm)), float(np.median(t_comp))
        diffs = np.array(t_norm) - np.array(t_comp)
        exposed = {"t_layer_ms": tn, "t_compute_only_ms": tcm,
                   "exposed_ms": tn - tcm, "exposed_pct": 100.0 * (tn - tcm) / tn,
                   "pair_diff_ms": {"median": float(np.median(diffs)), "min": float(diffs.min()),
                                    "max": float(diffs.max()), "p25": float(np.percentile(diffs, 25)),
                                    "p75": float(np.percentile(diffs, 75))},
                   "windows_layer_ms": t_norm, "windows_compute_only_ms": t_comp, "steps_per_window": wsteps,
                   "phases_compute_only_ms": {kk: round(v, 4) for kk, v in phases_co.items()},
                   "definition": "median T_layer - median T_compute_only over 10 alternating windows of "
                                 "graph-replayed steps (same kernels and tile order, peer buffers replaced by "
                                 "local ones, no barriers), max over ranks"}

    # ---- %globaltimer trace of graph-replayed steps (all ranks on one clock) ----
    gtrace = None
    if not args.no_graph:
        L.enable_stamps(True)
        step()
        sync_all()
        gst = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gst):
            step()
        steps_st = []
        for _ in range(10):
            gst.replay()
            sync_all()
            ph_ns, bars = L.read_stamps()
            steps_st.append((ph_ns, bars))
        L.enable_stamps(False)
        del gst
        for _ in range(2):
            step()
        sync_all()
        mine = {"rank": rank, "steps": [{"phases": p_, "barriers": {str(k_): v_ for k_, v_ in b_.items()}}
                                        for p_, b_ in steps_st]}
        if world > 1:
            allst = [None] * world
            dist.all_gather_object(allst, mine)
        else:
            allst = [mine]
        if rank == 0:
            from paper_2505_11432_b200.trace import stamp_summary
            gtrace = stamp_summary(allst)

    # ---- NCCL all-to-all baselines (standard unfused EP), same shapes ----
    nccl_ms = None
    nccl_gm_ms = None
    if not args.no_nccl_baseline and not injected and cfg.get("comm", "bf16") == "bf16":
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from nccl_moe_baseline import NcclMoEBaseline, NcclMoEGroupedBaseline
        g2 = torch.Generator(device="cuda").manual_seed(42)
        bw1 = (torch.randn(el, 2 * f, h, device="cuda", generator=g2) / h ** 0.5).bfloat16()
        bw2 = (torch.randn(el, h, f, device="cuda", generator=g2) / f ** 0.5).bfloat16()

        def time_baseline(cls):
            base = cls(Tr, h, f, E, k, n, rank, bw1, bw2, wr)
            for _ in range(2):
                base.step(x, dy)
            sync_all()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            nb = max(3, args.steps // 5)
            b0.record(stream)
            for _ in range(nb):
                base.step(x, dy)
            b1.record(stream)
            sync_all()
            tb = torch.tensor([b0.elapsed_time(b1) / nb], device="cuda")
            if world > 1:
                dist.all_reduce(tb, op=dist.ReduceOp.MAX)
            del base
            torch.cuda.empty_cache()
            return float(tb.item())
        nccl_ms = time_baseline(NcclMoEBaseline)
        try:
            nccl_gm_ms = time_baseline(NcclMoEGroupedBaseline)
        except Exception as e:  # noqa: BLE001
            nccl_gm_ms = None
            print("grouped_mm baseline failed:", str(e)[:200], file=sys.stderr)
        del bw1, bw2
        torch.cuda.empty_cache()

    # ---- per-phase device times (one instrumented step, same stream) ----
    L.enable_timing(True)
    phases = {}
    reps = 3
    for _ in range(reps):
        L.forward(None, y)
        L.backward(dy, dx, dw1, dw2, dwr)   # back to back: no idle gap between phases
        for kk, v in L.phase_times().items():
            phases[kk] = phases.get(kk, 0.0) + v / reps
    # memory-bound operators with the unfused dispatch (the reference's separate
    # scatter node) for their achieved HBM bandwidth
    membw = None
    if cfg.get("comm", "bf16") == "bf16" and cfg.get("gate", "before_fc2_in") == "before_fc2_in" \
            and args.ep_pattern == "a2a":
        fused_default = L.fused_dispatch()
        L.set_fused_dispatch(False)
        L.forward(None, y)
        L.backward(dy, dx, dw1, dw2, dwr)
        pu = L.phase_times()
        L.set_fused_dispatch(fused_default)
        rows_pad = routing_probe_rows(L, rank, el)
        hbm = load_peaks()["hbm"]
        rb = Tr * h * 2 + E * h * 2              # router: x + W_r
        sb = 2 * rows_pad * h * 2                # scatter: read rows + write permuted rows
        cb = (k + 1) * Tr * h * 2                # combine: k staged rows in + y out
        if world > 1 and "dispatch" in pu and pu["dispatch"] > 0:
            # NVLink pull rate of the standalone dispatch kernel (rows whose token
            # lives on a peer), against 900 GB/s per direction
            osr_u = L.routing()["out_source_rank"]
            rrows = int((osr_u != rank).sum().item())
            pull = rrows * h * 2 / (pu["dispatch"] * 1e6)
            nvlink_pull = {"remote_rows": rrows, "ms": pu["dispatch"], "GBps": pull, "frac_900": pull / 900.0}
        else:
            nvlink_pull = None
        membw = {kk: {"ms": pu[ph], "GBps": b / (pu[ph] * 1e6), "frac_hbm": b / (pu[ph] * 1e6) / hbm}
                 for kk, ph, b in (("router", "route", rb), ("scatter", "dispatch", sb), ("combine", "combine", cb))
                 if ph in pu and pu[ph] > 0}
    L.enable_timing(False)
    sync_all()

    # ---- end-to-end through the public API with host buffers ----
    # Every step uploads its own x and dy from pinned host memory and reads the
    # step's result back: its loss L = <y, dy> (the scalar whose gradient with
    # respect to y is the synthetic dy; bf16 dot on the device, 2 bytes to the
    # host). A second run also reads the whole dx back every step
    # (`with_dx_readback`). Copies run on a copy stream, double-buffered, so step
    # i+1's upload overlaps step i's backward and dx's readback overlaps the
    # weight-gradient GEMMs (dx_event fires before them).
    x_h = x.cpu().pin_memory()
    dy_h = dy.cpu().pin_memory()
    dx_h = torch.empty(Tr, h, dtype=torch.bfloat16).pin_memory()
    loss_h = torch.empty(2, dtype=torch.bfloat16).pin_memory()
    xb = [torch.empty_like(x) for _ in range(2)]
    dyb = [torch.empty_like(dy) for _ in range(2)]
    dxb = [torch.empty_like(dx) for _ in range(2)]
    loss_d = [torch.empty((), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    cs = torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    ev_dx = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def layer_step(b):
        L.forward(xb[b], y)
        L.backward(dyb[b], dxb[b], dw1, dw2, dwr, dx_event=ev_dx[b])
        torch.dot(y.view(-1), dyb[b].view(-1), out=loss_d[b])

    # The step's calls (forward + backward + loss on buffer set b) are captured
    # once per buffer set as a CUDA graph — what a fixed-shape training loop
    # does with these calls; the host copies stay outside, on the copy stream,
    # ordered by events (dx_event is recorded inside the graph).
    step_graphs = [None, None]
    if not args.no_graph:
        for b in range(2):
            xb[b].copy_(x)
            dyb[b].copy_(dy)
            layer_step(b)
            sync_all()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                layer_step(b)
            step_graphs[b] = gr
        sync_all()

    def e2e_run(nsteps, read_dx=False):
        with torch.cuda.stream(cs):
            xb[0].copy_(x_h, non_blocking=True)
            dyb[0].copy_(dy_h, non_blocking=True)
            ev_in[0].record(cs)
        for i in range(nsteps):
            b = i % 2
            stream.wait_event(ev_in[b])
            if i >= 2:
                stream.wait_event(ev_out[b])   # buffer set b's results drained to the host
            if step_graphs[b] is not None:
                step_graphs[b].replay()
            else:
                L.forward(xb[b], y)
            if i + 1 < nsteps:
                with torch.cuda.stream(cs):
                    if i >= 1:
                        cs.wait_event(ev_free[1 - b])
                    xb[1 - b].copy_(x_h, non_blocking=True)
                    dyb[1 - b].copy_(dy_h, non_blocking=True)
                    ev_in[1 - b].record(cs)
            if step_graphs[b] is None:
                L.backward(dyb[b], dxb[b], dw1, dw2, dwr, dx_event=ev_dx[b])
                torch.dot(y.view(-1), dyb[b].view(-1), out=loss_d[b])
            ev_free[b].record(stream)
            ev_done[b].record(stream)
            with torch.cuda.stream(cs):
                if read_dx:
                    cs.wait_event(ev_dx[b])
                    dx_h.copy_(dxb[b], non_blocking=True)
                cs.wait_event(ev_done[b])
                loss_h[b].copy_(loss_d[b], non_blocking=True)
                ev_out[b].record(cs)
        stream.wait_stream(cs)

    def e2e_time(read_dx):
        e2e_run(2, read_dx)
        sync_all()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_run(args.steps, read_dx)
        e1.record(stream)
        sync_all()
        te = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return float(te.item())

    e2e_ms = e2e_time(False)
    e2e_dx_ms = e2e_time(True)
    # the same host copies alone (every rank at once, no compute): the floor the
    # host link puts under the e2e step (uploads, + the dx readback)
    def copies_only(read_dx):
        sync_all()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(cs):
            c0.record(cs)
            for i in range(args.steps):
                xb[i % 2].copy_(x_h, non_blocking=True)
                dyb[i % 2].copy_(dy_h, non_blocking=True)
                if read_dx:
                    dx_h.copy_(dxb[i % 2], non_blocking=True)
            c1.record(cs)
        sync_all()
        tc = torch.tensor([c0.elapsed_time(c1) / args.steps], device="cuda")
        if world > 1:
            dist.all_reduce(tc, op=dist.ReduceOp.MAX)
        return float(tc.item())

    copy_only_ms = copies_only(False)
    copy_only_dx_ms = copies_only(True)

    rt = L.routing()
    cnt = rt["per_expert_counts"].cpu().tolist()[rank * el:(rank + 1) * el]
    # exact NVLink volume of this rank's fused exchanges (rows whose source
    # token lives on another rank): dispatch pull + combine push, fwd and bwd
    nvlink = None
    if n > 1:
        osr = rt["out_source_rank"].cpu()
        remote = osr != rank
        remote_rows = int(remote.sum().item())
        # dispatch dedup: a token with several experts on this rank is pulled once
        # (layer.cu `dedup`; the gate-after backward pulls every row)
        tok = rt["row_map_in"].cpu()[remote] // L.k
        remote_tokens = int(torch.unique(tok).numel())
        dedup = os.environ.get("MOE_NO_DISPATCH_DEDUP") is None and L.k > 1 and L.E // n > 1
        pulled_fwd = remote_tokens if dedup else remote_rows
        pulled_bwd = remote_rows if cfg.get("gate") == "after_fc2_out" else pulled_fwd
        bpe = 1 if cfg.get("comm", "bf16") == "fp8" else 2
        fwd_b = (pulled_fwd + remote_rows) * h * bpe  # dispatch x in + combine y out
        bwd_b = (pulled_bwd + remote_rows) * h * bpe  # dispatch dy in + combine dx out
        if args.ep_pattern == "ag_rs":
            # all-gather of every peer token row in; one pre-reduced partial per
            # (remote token, this rank) out (sparse reduce-scatter)
            ex_all = rt["experts"].cpu()
            served = ((ex_all // el) == rank).any(1)
            own = (torch.arange(ex_all.shape[0]) // Tr) == rank
            rs_rows = int((served & ~own).sum().item())
            fwd_b = ((n - 1) * Tr + rs_rows) * h * bpe
            bwd_b = fwd_b
            pulled_fwd = (n - 1) * Tr
        measured = None
        allm = [None] * world
        dist.all_gather_object(allm, nvl_meas)
        if all(m_ is not None for m_ in allm):
            tx_max = max(m_[0] for m_ in allm)
            rx_max = max(m_[1] for m_ in allm)
            measured = {"source": "NVML NVLINK_THROUGHPUT_DATA_TX/RX over the timed region, per rank per step",
                        "tx_bytes_per_step_per_rank": [m_[0] for m_ in allm],
                        "rx_bytes_per_step_per_rank": [m_[1] for m_ in allm],
                        "max_GBps_tx": tx_max / (ms / 1000.0) / 1e9, "max_GBps_rx": rx_max / (ms / 1000.0) / 1e9,
                        "frac_900_over_step": max(tx_max, rx_max) / (ms / 1000.0) / 900e9}
        if measured is None:
            measured = {"unavailable": "NVML NVLink throughput counters return NOT_SUPPORTED on this pool "
                                       "(scripts/nvml_nvlink_probe.py); ncu NVLink metrics need one profiled "
                                       "process per rank, which hangs the flag barriers"}
        # the link rate each fused kernel needs: its NVLink bytes over its own busy
        # time in the graph-replayed steps (max over ranks), against 900 GB/s
        per_phase = None
        busy = (gtrace or {}).get("summary", {}).get("phases_busy_ms") if isinstance(gtrace, dict) else None
        if busy:
            ph_bytes = {"fc1": pulled_fwd * h * bpe, "fc2": remote_rows * h * bpe,
                        "fc2_dgrad": pulled_bwd * h * bpe, "fc1_dgrad": remote_rows * h * bpe}
            if args.ep_pattern == "ag_rs":
                ph_bytes = {"fc1": (n - 1) * Tr * h * bpe, "fc2": rs_rows * h * bpe,
                            "fc2_dgrad": (n - 1) * Tr * h * bpe, "fc1_dgrad": rs_rows * h * bpe}
            per_phase = {ph: {"bytes": b, "busy_ms": busy.get(ph),
                              "GBps": (b / (busy[ph] / 1000.0) / 1e9) if busy.get(ph) else None,
                              "frac_900": (b / (busy[ph] / 1000.0) / 900e9) if busy.get(ph) else None}
                         for ph, b in ph_bytes.items()}
        nvlink = {"measured_nvml": measured, "per_fused_kernel": per_phase, "remote_rows": remote_rows, "remote_tokens": remote_tokens, "rows_pulled": pulled_fwd,
                  "bytes_per_step": fwd_b + bwd_b,
                  "link_GBps_if_spread_over_step": (fwd_b + bwd_b) / (ms / 1000.0) / 1e9,
                  "link_time_ms_at_770GBps": (fwd_b + bwd_b) / 770e9 * 1000.0,
                  "note": "bytes per direction per rank; overlapped inside fc1/fc2/fc2-dgrad/fc1-dgrad"}
    # ---- the six expert GEMMs vs torch._grouped_mm / per-expert cuBLAS, same shapes ----
    gemm_cmp = None
    if n == 1 and not args.no_gemm_compare and cfg.get("comm", "bf16") == "bf16":
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from cublas_gemm_baseline import compare_gemms
        gemm_cmp = compare_gemms(h, f, [int(c) for c in cnt])
        fused = {"fc1": "fc1", "fc2": "fc2", "fc2_dgrad": "fc2_dgrad", "fc1_dgrad": "fc1_dgrad",
                 "fc2_wgrad": "fc2_wgrad", "fc1_wgrad": "fc1_wgrad"}
        gemm_cmp["layer_fused_ms"] = {kk: round(phases.get(v, float("nan")), 4) for kk, v in fused.items()}
        torch.cuda.empty_cache()
    pad = layer_pad(L)
    routing_info = {"local_rows": int(sum(cnt)), "padded_rows": int(sum((c + pad - 1) // pad * pad for c in cnt)),
                    "row_padding": pad,
                    "max_expert_rows": int(max(cnt)), "min_expert_rows": int(min(cnt))}
    if rank == 0:
        peaks = load_peaks()
        rows = Tr * k * n  # expert rows processed per rank (uniform expectation)
        rows_local = Tr * k  # per rank in expectation (weak scaling)
        fc1_flops = 2.0 * rows_local * h * 2 * f
        fc1_ms = phases.get("fc1", float("nan"))
        achieved = fc1_flops / (fc1_ms / 1000.0) / 1e12
        total_flops = 3.0 * rows_local * 6.0 * h * f  # fwd+bwd expert FFN
        traffic = None
        try:  # DRAM bytes per fc1 launch from the committed ncu capture (same workload)
            with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as fh:
                if cfg["workload"].startswith("mixtral-8x7b-moe-layer-fwd+bwd") and n == 1:
                    traffic = json.load(fh)["kernels"]["fc1"]["traffic_bytes"]
        except Exception:
            traffic = None
        # fc1's bound: tensor time vs HBM time of its algorithmic bytes (this rank's
        # W1 once, the permuted rows in, fc1_out + fc2_in out). Fine-grained experts
        # on few GPUs (DeepSeek shape at n = 1: 15 GB of W1) are HBM-bound.
        fc1_bytes = el * 2 * f * h * 2 + rows_local * h * 2 + rows_local * 3 * f * 2
        t_tc, t_hbm = fc1_flops / (peaks["bf16_sus"] * 1e12), fc1_bytes / (peaks["hbm"] * 1e9)
        # step: expert FLOPs vs weights read twice (fwd, dgrad) + weight grads written
        # + activations (x, fc1_out, fc2_in, dy, dfc1 streams)
        step_bytes = 3 * el * 3 * f * h * 2 + rows_local * (4 * h + 8 * f) * 2
        st_tc, st_hbm = total_flops / (peaks["bf16_sus"] * 1e12), step_bytes / (peaks["hbm"] * 1e9)
        if t_hbm > t_tc:
            gbs = fc1_bytes / (fc1_ms / 1000.0) / 1e9
            roof = {"bound": "hbm", "kernel": "fc1 grouped GEMM (tcgen05) + fused SwiGLU",
                    "achieved": gbs, "peak": peaks["hbm"], "unit": "GB/s", "frac": gbs / peaks["hbm"],
                    "traffic": traffic, "algorithmic_bytes": fc1_bytes, "peak_kind": f"HBM ({peaks['src']})"}
        else:
            roof = {"bound": "tensor", "kernel": "fc1 grouped GEMM (tcgen05) + fused SwiGLU",
                    "achieved": achieved, "peak": peaks["bf16_sus"], "unit": "TFLOP/s",
                    "frac": achieved / peaks["bf16_sus"], "traffic": traffic,
                    "algorithmic_bytes": fc1_bytes, "peak_kind": f"bf16 sustained ({peaks['src']})"}
        # n > 1: NVLink bytes of this rank's fused exchanges at the measured link rate
        st_link = (nvlink["bytes_per_step"] / 770e9) if nvlink else 0.0
        bounds = {"tensor": st_tc, "hbm": st_hbm, "nvlink": st_link}
        sb_name = max(bounds, key=bounds.get)
        roof.update({"step_bound": sb_name,
                     "step_roofline_ms": 1000 * bounds[sb_name],
                     "step_frac": 1000 * bounds[sb_name] / ms,
                     "step_bound_ms": {kk: round(1000 * v, 4) for kk, v in bounds.items()},
                     "step_tflops": total_flops / (ms / 1000.0) / 1e12})
        line = {
            "metric": "moe_layer_fwd_bwd_tokens_per_s", "value": value, "unit": "tokens/s",
            "n_gpus": n, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": ("synthetic (random-init weights, N(0,0.25) tokens; " +
                     ("injected Zipf routing from the reference's simulate_routing)" if injected else "learned router)")),
            "config": {"workload": cfg["workload"], "hidden": h, "ffn_hidden": f, "num_experts": E,
                       "top_k": k, "tokens_per_rank": Tr, "global_tokens": Tr * n,
                       "parallelism": f"ep{n}", "comm_format": cfg.get("comm", "bf16"),
                       "gate_order": cfg.get("gate", "before_fc2_in"), "ep_pattern": args.ep_pattern,
                       "remat": "off" if args.no_remat else "selective",
                       "dispatch": "fused into fc1 / fc2-dgrad" if L.fused_dispatch() else "separate scatter kernel",
                       "l2": "inputs larger than L2 (expert weights >= 2.8 GB/layer)"},
            "roofline": roof,
            "phases_ms": {kk: round(v, 4) for kk, v in phases.items()},
            "routing_rank0": routing_info,
            "memory_bound_ops": membw,
            "exposed_comm": exposed,
            "graph_trace": None if gtrace is None else gtrace["summary"],
            # expert-GEMM throughput inside the graph-replayed steps: this rank's real
            # rows over each GEMM's busy time (max over ranks), vs the sustained peak
            "gemm_tflops_in_step": None if gtrace is None else {
                ph: {"busy_ms": gtrace["summary"]["phases_busy_ms"].get(ph),
                     "tflops": fl / (gtrace["summary"]["phases_busy_ms"][ph] / 1000.0) / 1e12,
                     "frac_sustained": fl / (gtrace["summary"]["phases_busy_ms"][ph] / 1000.0) / 1e12
                                       / load_peaks()["bf16_sus"]}
                for ph, fl in (("fc1", 2.0 * routing_info["local_rows"] * h * 2 * f),
                               ("fc2", 2.0 * routing_info["local_rows"] * f * h),
                               ("fc2_dgrad", 2.0 * routing_info["local_rows"] * h * f),
                               ("fc1_dgrad", 2.0 * routing_info["local_rows"] * 2 * f * h),
                               ("fc2_wgrad", 2.0 * routing_info["local_rows"] * h * f),
                               ("fc1_wgrad", 2.0 * routing_info["local_rows"] * 2 * f * h))
                if gtrace["summary"]["phases_busy_ms"].get(ph)},
            "nvlink": nvlink,
            "gemm_vs_cublas": gemm_cmp,
            "nvlink_dispatch_pull": nvlink_pull if membw is not None else None,
            "nccl_a2a_cublas_baseline": None if nccl_ms is None else {
                "ms_per_step": nccl_ms, "tokens_per_s": n * Tr / (nccl_ms / 1000.0),
                "speedup_of_fused": nccl_ms / ms,
                "what": "standard EP: NCCL all_to_all_single dispatch/combine + per-expert cuBLAS (torch) fwd+bwd"},
            "nccl_a2a_grouped_mm_baseline": None if nccl_gm_ms is None else {
                "ms_per_step": nccl_gm_ms, "tokens_per_s": n * Tr / (nccl_gm_ms / 1000.0),
                "speedup_of_fused": nccl_gm_ms / ms,
                "what": "NCCL all_to_all_single dispatch/combine + one torch._grouped_mm (CUTLASS) per expert "
                        "GEMM, bf16 SwiGLU / gate backward in torch ops"},
            "clocks": clk,
            "gpu_launches": int(launches),
            "gpu_launches_per_step": int(per_step_launches),
            "launch_mode": "eager" if args.no_graph else "cuda_graph",
            "e2e": {"value": n * Tr / (e2e_ms / 1000.0), "unit": "tokens/s",
                    "h2d_bytes_per_step": 2 * Tr * h * 2, "d2h_bytes_per_step": 2,
                    "ms_per_step": e2e_ms, "host_copies_only_ms_per_step": copy_only_ms,
                    "mode": ("MoELayer.forward/backward (+ the step's loss <y, dy>) captured as one CUDA graph "
                             "per buffer set; x, dy uploaded from pinned host memory and the loss read back "
                             "every step on a copy stream"
                             if not args.no_graph else "eager MoELayer.forward/backward calls; same copies"),
                    "with_dx_readback": {"value": n * Tr / (e2e_dx_ms / 1000.0), "ms_per_step": e2e_dx_ms,
                                         "d2h_bytes_per_step": Tr * h * 2 + 2,
                                         "host_copies_only_ms_per_step": copy_only_dx_ms}},
        }
        if n == 1 and not args.no_cpu_baseline:
            try:
                r = cpu_reference_step(cfg, 1, max_dense_tokens=256)  # warm (pages, BLAS threads)
                r = cpu_reference_step(cfg, 1)
                line["cpu_baseline"] = {"value": r["value"], "unit": "tokens/s", "cores": r["cores"],
                                        "kind": r["kind"], "sample": _cpu_sample_text(r)}
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
            if not args.no_integer_compare:
                try:
                    sys.path.insert(0, os.path.join(ROOT, "scripts"))
                    from integer_path_bench import compare as integer_compare
                    line["reference_integer_path"] = integer_compare()
                except Exception as e:  # noqa: BLE001
                    line["reference_integer_path"] = {"error": str(e)[:200]}
        if args.trace:
            from paper_2505_11432_b200.trace import write_stamp_trace, write_trace
            if gtrace is not None:
                write_stamp_trace(args.trace, gtrace, Tr * k, h, f,
                                  exposed["exposed_ms"] / 1000.0 if exposed else None)
            else:
                write_trace(args.trace, phases, Tr * k, h, f,
                            exposed["exposed_ms"] / 1000.0 if exposed else None)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_f32(args, cfg):
    """configs[0]: the fp32 layer forward (router, capacity drop, permutation,
    FFMA expert GEMMs, SwiGLU, combine) on one GPU, against the FFMA roofline
    (148 SMs x 128 fp32 lanes x 2 FLOP x SM clock)."""
    import torch
    from paper_2505_11432_b200 import launch_count, launch_count_reset, ops
    torch.cuda.set_device(0)
    h, f, E, k, T = cfg["hidden"], cfg["ffn_hidden"], cfg["num_experts"], cfg["top_k"], cfg["tokens_per_rank"]
    g = torch.Generator(device="cuda").manual_seed(42)
    w1 = torch.randn(E, 2 * f, h, device="cuda", generator=g) / h ** 0.5
    w2 = torch.randn(E, h, f, device="cuda", generator=g) / f ** 0.5
    wr = torch.randn(E, h, device="cuda", generator=g) / h ** 0.5
    x = torch.randn(T, h, device="cuda", generator=g) * 0.5
    for _ in range(args.warmup):
        ops.ffn_forward_f32(x, w1, w2, wr, k)
    torch.cuda.synchronize()
    launch_count_reset()
    ops.ffn_forward_f32(x, w1, w2, wr, k)
    torch.cuda.synchronize()
    per_step = launch_count()
    clocks = ClockSampler(0)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        ops.ffn_forward_f32(x, w1, w2, wr, k)
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    # e2e: host x in, host y out, through the public operator
    xh = x.cpu().pin_memory()
    yh = torch.empty(T, h, dtype=torch.float32).pin_memory()
    e0.record()
    for _ in range(args.steps):
        xd = xh.to("cuda", non_blocking=True)
        y = ops.ffn_forward_f32(xd, w1, w2, wr, k)[0]
        yh.copy_(y, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    flops = 2.0 * T * k * h * 2 * f + 2.0 * T * k * f * h + 2.0 * T * h * E
    mhz = clk["sm_mhz"] or 1965.0
    ffma_peak = 148 * 128 * 2 * mhz * 1e6 / 1e12
    ffma_mode = os.environ.get("MOE_F32_FFMA") is not None
    tc_peak = load_peaks()["bf16_sus"] / 6.0   # bf16x6: six bf16 MMAs per fp32 product
    line = {
        "metric": "moe_layer_fwd_tokens_per_s", "value": T / (ms / 1000.0), "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (random-init weights)",
        "config": {"workload": cfg["workload"], "hidden": h, "ffn_hidden": f, "num_experts": E, "top_k": k,
                   "tokens": T, "l2": "weights 277 MB > L2"},
        "roofline": ({"bound": "ffma", "achieved": flops / (ms / 1000.0) / 1e12, "peak": ffma_peak,
                      "unit": "TFLOP/s", "frac": flops / (ms / 1000.0) / 1e12 / ffma_peak, "traffic": None,
                      "peak_kind": "derived FFMA peak at the measured median SM clock (148 x 128 x 2 x clock)",
                      "roofline_ms": flops / (ffma_peak * 1e12) * 1000.0} if ffma_mode else
                     {"bound": "tensor", "achieved": flops / (ms / 1000.0) / 1e12, "peak": tc_peak,
                      "unit": "TFLOP/s (fp32 algorithmic)", "frac": flops / (ms / 1000.0) / 1e12 / tc_peak,
                      "traffic": None,
                      "peak_kind": "bf16 sustained peak / 6 (the bf16x6 split runs six bf16 MMAs per fp32 "
                                   "product term; measured peak)",
                      "roofline_ms": flops / (tc_peak * 1e12) * 1000.0,
                      "vs_ffma_roofline": {"ffma_peak": ffma_peak,
                                           "ffma_roofline_ms": flops / (ffma_peak * 1e12) * 1000.0}}),
        "gemm_path": "FFMA grouped GEMMs" if ffma_mode else "bf16x6 tcgen05 grouped GEMMs (fp32-accurate split)",
        "e2e": {"value": T / (e2e_ms / 1000.0), "unit": "tokens/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": T * h * 4, "d2h_bytes_per_step": T * h * 4},
        "clocks": clk, "gpu_launches": int(per_step * args.steps), "gpu_launches_per_step": int(per_step),
    }
    print(json.dumps(line), flush=True)


def run_attn(args, cfg):
    """configs[3]: fused AG-GEMM (QKV) + GEMM-RS (out-proj) at TP = n, with the
    NCCL all-gather / reduce-scatter + cuBLAS baseline timed in the same run."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2505_11432_b200 import launch_count, launch_count_reset
    from paper_2505_11432_b200.attn import AttnProjections
    n, s_len, h, m = world, cfg["seq"], cfg["hidden"], cfg["gqa"]
    nq = h * (m + 2) // m // n                 # h (1 + 2/m) / n  (graph.cpp:163-165)
    dh, sr = h // n, s_len // n
    g = torch.Generator(device="cuda").manual_seed(3 + rank)
    wqkv = (torch.randn(nq, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
    wout = (torch.randn(h, dh, device="cuda", generator=g) / dh ** 0.5).bfloat16()
    x = (torch.randn(sr, h, device="cuda", generator=g) * 0.5).bfloat16()
    o = (torch.randn(s_len, dh, device="cuda", generator=g) * 0.5).bfloat16()
    A = AttnProjections(s_len, h, nq, n, rank)
    A.set_weights(wqkv, wout)
    if n > 1:
        A.connect()
    A.input_buffer.copy_(x)
    qkv = torch.empty(s_len, nq, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(sr, h, dtype=torch.bfloat16, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        A.ag_gemm(None, qkv)
        A.gemm_rs(o, y)

    def sync_all():
        torch.cuda.synchronize()
        if n > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        sync_all()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            fn()
        e1.record(stream)
        sync_all()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
        if n > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    launch_count_reset()
    step()
    per_step = launch_count()
    nvl = None
    if n > 1:
        try:
            nvl = NvlinkCounters(local)
            if not nvl.probe():
                nvl = None
        except Exception:  # noqa: BLE001
            nvl = None
    nv0 = nvl.read() if nvl else None
    clocks = ClockSampler(local)
    clocks.start()
    ms = timed(step)
    clk = clocks.stop()
    nv_step = None
    if nvl:
        nv1 = nvl.read()
        nsteps = args.steps + args.warmup
        nv_step = [(nv1[0] - nv0[0]) / nsteps, (nv1[1] - nv0[1]) / nsteps]
    nv_all = None
    if n > 1:
        nv_all = [None] * n
        dist.all_gather_object(nv_all, nv_step)
    ms_ag = timed(lambda: A.ag_gemm(None, qkv))
    ms_rs_only = timed(lambda: A.gemm_rs(o, y))
    # NCCL + cuBLAS baseline for the same math
    xg = torch.empty(s_len, h, dtype=torch.bfloat16, device="cuda")
    part = torch.empty(s_len, h, dtype=torch.bfloat16, device="cuda")

    def nccl_step():
        if n > 1:
            dist.all_gather_into_tensor(xg, x)
        else:
            xg.copy_(x)
        torch.matmul(xg, wqkv.T, out=qkv)
        torch.matmul(o, wout.T, out=part)
        if n > 1:
            dist.reduce_scatter_tensor(y, part)
        else:
            y.copy_(part)
    ms_nccl = timed(nccl_step)
    if rank == 0:
        peaks = load_peaks()
        flops = 2.0 * s_len * h * nq + 2.0 * s_len * dh * h
        link_bytes = 2.0 * (n - 1) / n * s_len * h * 2 if n > 1 else 0.0
        t_tensor = flops / (peaks["bf16"] * 1e12)
        t_link = link_bytes / 770e9
        line = {
            "metric": "sp_attention_projection_pair_tokens_per_s", "value": s_len / (ms / 1000.0),
            "unit": "tokens/s", "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": cfg["workload"], "hidden": h, "seq": s_len, "gqa_ratio": m,
                       "qkv_cols_per_rank": nq, "parallelism": f"tp{n}-sp{n}"},
            "roofline": {"bound": "nvlink" if t_link > t_tensor else "tensor",
                         "target_ms": 1000 * max(t_tensor, t_link), "achieved_ms": ms,
                         "frac": 1000 * max(t_tensor, t_link) / ms,
                         "peak": "bf16 %.1f TF (measured burst), NVLink 770 GB/s/dir (measured ref.)" % peaks["bf16"]},
            "ag_gemm_ms": ms_ag, "gemm_rs_ms": ms_rs_only,
            "per_op_roofline": {
                "ag_gemm": {"target_ms": 1000 * max(2.0 * s_len * h * nq / (peaks["bf16"] * 1e12),
                                                    (n - 1) / n * s_len * h * 2 / 770e9 if n > 1 else 0.0),
                            "achieved_ms": ms_ag},
                "gemm_rs": {"target_ms": 1000 * max(2.0 * s_len * dh * h / (peaks["bf16"] * 1e12),
                                                    (n - 1) / n * s_len * h * 2 / 770e9 if n > 1 else 0.0),
                            "achieved_ms": ms_rs_only}},
            "nvlink_measured_nvml": None if not nv_all or any(v is None for v in nv_all) else {
                "tx_bytes_per_step_per_rank": [v[0] for v in nv_all], "rx_bytes_per_step_per_rank": [v[1] for v in nv_all],
                "algorithmic_bytes_per_step_per_rank": 2.0 * (n - 1) / n * s_len * h * 2,
                "GBps_rx_max": max(v[1] for v in nv_all) / (ms / 1000.0) / 1e9},
            "nccl_cublas_baseline_ms": ms_nccl, "speedup_vs_nccl_baseline": ms_nccl / ms,
            "clocks": clk, "gpu_launches": per_step * args.steps, "launch_mode": "eager",
            "e2e": None,
        }
        print(json.dumps(line), flush=True)
    if n > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_ulysses(args, cfg):
    """§8f row 3: fused GEMM+A2A (QKV) and A2A+GEMM (out-proj) at SP = n, with
    the cuBLAS + NCCL all_to_all baseline (incl. its layout permutes) timed in
    the same run."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2505_11432_b200 import launch_count, launch_count_reset
    from paper_2505_11432_b200.ulysses import UlyssesProjections
    n, s_len, h, m = world, cfg["seq"], cfg["hidden"], cfg["gqa"]
    nqkv = h * (m + 2) // m                    # h (1 + 2/m)  (graph.cpp:163-165)
    sr, cpo, dh = s_len // n, nqkv // n, h // n
    g = torch.Generator(device="cuda").manual_seed(3)
    wqkv = (torch.randn(nqkv, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
    wout = (torch.randn(h, h, device="cuda", generator=g) / h ** 0.5).bfloat16()
    g.manual_seed(11 + rank)
    x = (torch.randn(sr, h, device="cuda", generator=g) * 0.5).bfloat16()
    o = (torch.randn(s_len, dh, device="cuda", generator=g) * 0.5).bfloat16()
    U = UlyssesProjections(s_len, h, nqkv, n, rank)
    U.set_weights(wqkv, wout)
    if n > 1:
        U.connect()
    U.attn_out.copy_(o)
    y = torch.empty(sr, h, dtype=torch.bfloat16, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        U.qkv_a2a(x)
        U.a2a_out_proj(None, y)

    def sync_all():
        torch.cuda.synchronize()
        if n > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        sync_all()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            fn()
        e1.record(stream)
        sync_all()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
        if n > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    launch_count_reset()
    step()
    per_step = launch_count()
    clocks = ClockSampler(local)
    clocks.start()
    ms = timed(step)
    clk = clocks.stop()
    ms_qkv = timed(lambda: U.qkv_a2a(x))
    base = None
    if not args.no_nccl_baseline:
        qkv_loc = torch.empty(sr, nqkv, dtype=torch.bfloat16, device="cuda")
        send = torch.empty(n, sr, cpo, dtype=torch.bfloat16, device="cuda")
        recv = torch.empty(s_len, cpo, dtype=torch.bfloat16, device="cuda")
        orecv = torch.empty(n, sr, dh, dtype=torch.bfloat16, device="cuda")
        oseq = torch.empty(sr, h, dtype=torch.bfloat16, device="cuda")

        def nccl_step():
            torch.matmul(x, wqkv.T, out=qkv_loc)
            send.copy_(qkv_loc.view(sr, n, cpo).transpose(0, 1))
            if n > 1:
                dist.all_to_all_single(recv, send.view(-1, cpo))
                dist.all_to_all_single(orecv.view(-1, dh), o)
            else:
                recv.copy_(send.view(-1, cpo))
                orecv.view(-1, dh).copy_(o)
            oseq.view(sr, n, dh).copy_(orecv.transpose(0, 1))
            torch.matmul(oseq, wout.T, out=y)
        base = timed(nccl_step)
    if rank == 0:
        peaks = load_peaks()
        flops = 2.0 * sr * h * nqkv + 2.0 * sr * h * h
        link_bytes = (n - 1) / n * (s_len * cpo + s_len * dh) * 2 if n > 1 else 0.0   # into each rank
        t_tensor = flops / (peaks["bf16"] * 1e12)
        t_link = link_bytes / 770e9
        line = {
            "metric": "ulysses_attention_projection_pair_tokens_per_s", "value": s_len / (ms / 1000.0),
            "unit": "tokens/s", "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": cfg["workload"], "hidden": h, "seq": s_len, "gqa_ratio": m,
                       "qkv_cols": nqkv, "parallelism": f"sp{n}"},
            "roofline": {"bound": "nvlink" if t_link > t_tensor else "tensor",
                         "target_ms": 1000 * max(t_tensor, t_link), "achieved_ms": ms,
                         "frac": 1000 * max(t_tensor, t_link) / ms,
                         "peak": "bf16 %.1f TF (measured burst), NVLink 770 GB/s/dir (measured ref.)" % peaks["bf16"]},
            "qkv_gemm_a2a_ms": ms_qkv, "a2a_out_proj_gemm_ms": ms - ms_qkv,
            "nccl_cublas_baseline_ms": base, "speedup_vs_nccl_baseline": (base / ms) if base else None,
            "clocks": clk, "gpu_launches": per_step * args.steps, "launch_mode": "eager", "e2e": None,
        }
        print(json.dumps(line), flush=True)
    if n > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_dp(args, cfg):
    """§8f row 4: compressed DP reduce-scatter (bf16 all-to-all + wide local
    reduce, in place) and bf16 all-gather, beside NCCL's fp32 / bf16
    reduce-scatter and bf16 all-gather of the same buffer."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2505_11432_b200 import launch_count, launch_count_reset
    from paper_2505_11432_b200.dp import DpGradSync
    n, count = world, cfg["count"]
    S = count // n
    D = DpGradSync(count, n, rank)
    if n > 1:
        D.connect()
    g = torch.Generator(device="cuda").manual_seed(5 + rank)
    D.grad.copy_(torch.randn(count, device="cuda", generator=g) * 1e-3)
    upd = torch.randn(S, device="cuda", generator=g)
    full = torch.empty(count, dtype=torch.bfloat16, device="cuda")
    stream = torch.cuda.current_stream()

    def sync_all():
        torch.cuda.synchronize()
        if n > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        sync_all()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            fn()
        e1.record(stream)
        sync_all()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
        if n > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    launch_count_reset()
    D.reduce_scatter()
    per_step = launch_count()
    clocks = ClockSampler(local)
    clocks.start()
    # the buffer holds whatever the previous call left (finite floats): the
    # timing does not depend on the values
    ms_rs = timed(lambda: D.reduce_scatter())
    clk = clocks.stop()
    ms_ag = timed(lambda: D.all_gather_bf16(upd, full))
    base = {}
    if n > 1 and not args.no_nccl_baseline:
        g32 = torch.randn(count, device="cuda", generator=g)
        s32 = torch.empty(S, device="cuda")
        g16, s16 = g32.bfloat16(), torch.empty(S, dtype=torch.bfloat16, device="cuda")
        base["nccl_fp32_reduce_scatter_ms"] = timed(lambda: dist.reduce_scatter_tensor(s32, g32))
        base["nccl_bf16_reduce_scatter_ms"] = timed(lambda: dist.reduce_scatter_tensor(s16, g16))
        base["nccl_bf16_all_gather_ms"] = timed(lambda: dist.all_gather_into_tensor(full, s16))
        del g32, g16
    if rank == 0:
        peaks = load_peaks()
        wire = 2.0 * (n - 1) / n * count          # bf16 bytes into each rank per collective
        # cast r+w, a2a reads, shard write (n = 1: one in-place read + write)
        hbm = 8.0 * count if n == 1 else 4.0 * count + 2.0 * count + 2.0 * count + 4.0 * S
        t_link = wire / 770e9
        t_hbm = hbm / (peaks["hbm"] * 1e9)
        bound = "nvlink" if t_link > t_hbm else "hbm"
        line = {
            "metric": "dp_grad_sync_fp32_bytes_per_s", "value": count * 4 / (ms_rs / 1000.0) / 1e9,
            "unit": "GB/s (fp32 gradient bytes reduce-scattered per rank)", "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_rs, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16 wire / fp64 reduce / fp32 out",
            "data": "synthetic",
            "config": {"workload": cfg["workload"], "count": count, "dp": n, "shard": S,
                       "inputs": "buffer > L2 (705 MB fp32)"},
            "roofline": {"bound": bound, "target_ms": 1000 * max(t_link, t_hbm), "achieved_ms": ms_rs,
                         "frac": 1000 * max(t_link, t_hbm) / ms_rs,
                         "peak": "NVLink 770 GB/s/dir (measured ref.), HBM %.0f GB/s" % peaks["hbm"]},
            "reduce_scatter_ms": ms_rs, "all_gather_bf16_ms": ms_ag, **base,
            "clocks": clk, "gpu_launches": per_step * args.steps, "launch_mode": "eager", "e2e": None,
        }
        if "nccl_fp32_reduce_scatter_ms" in base:
            line["speedup_vs_nccl_fp32_rs"] = base["nccl_fp32_reduce_scatter_ms"] / ms_rs
        print(json.dumps(line), flush=True)
    if n > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels eagerly instead of one CUDA graph per step")
    ap.add_argument("--no-nccl-baseline", action="store_true")
    ap.add_argument("--no-integer-compare", action="store_true",
                    help="skip the full-shape reference integer path vs device kernels block (N=1)")
    ap.add_argument("--no-gemm-compare", action="store_true",
                    help="skip the per-GEMM torch._grouped_mm / cuBLAS comparison (N=1)")
    ap.add_argument("--ep-pattern", default="a2a", choices=["a2a", "ag_rs"],
                    help="EP dispatch/combine pattern (commcost.hpp:81): needed-row pulls + per-slot pushes, "
                         "or all-gather + local scatter and per-rank pre-reduced reduce-scatter")
    ap.add_argument("--no-remat", action="store_true",
                    help="RematPolicy::off (reference --no-remat): keep the forward's fc2_in for the fc2 wgrad")
    ap.add_argument("--trace", default=None, help="write the measured per-phase timeline (reference trace schema)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.config == "ulysses":
        run_ulysses(args, cfg)
    elif args.config == "dp":
        run_dp(args, cfg)
    elif args.config == "attn":
        run_attn(args, cfg)
    elif args.config == "small_f32":
        run_f32(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
