"""Probe (not the product): steady-state throughput, SM clock and board power
of our grouped GEMM vs torch._grouped_mm at the fc1 / fc2-dgrad shapes
(Mixtral, 1024 rows per expert), each run back to back for ~1.5 s while NVML
is sampled every 10 ms. Under the power cap the GEMM with the lower energy per
FLOP holds the higher clock.
Usage: python scripts/gemm_power_probe.py"""
import json
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from paper_2505_11432_b200 import ops  # noqa: E402


def sampler(stop, out):
    import pynvml as N
    N.nvmlInit()
    hd = N.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    while not stop.is_set():
        out.append((N.nvmlDeviceGetPowerUsage(hd) / 1000.0, N.nvmlDeviceGetClockInfo(hd, N.NVML_CLOCK_SM)))
        time.sleep(0.01)


def run(fn, flops, seconds=1.5):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.time()
    n = 0
    while time.time() - t0 < 0.3:
        fn(); n += 1
    torch.cuda.synchronize()
    per = 0.3 / max(n, 1)
    reps = max(10, int(seconds / per))
    stop, samp = threading.Event(), []
    th = threading.Thread(target=sampler, args=(stop, samp))
    th.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    stop.set(); th.join()
    ms = a.elapsed_time(b) / reps
    samp = samp[len(samp) // 5:]   # drop the ramp
    pw = sorted(s[0] for s in samp); ck = sorted(s[1] for s in samp)
    return {"tflops": round(flops / ms / 1e9, 1), "ms": round(ms, 4), "power_w": pw[len(pw) // 2],
            "sm_mhz": ck[len(ck) // 2], "tflop_per_joule": round(flops / ms / 1e9 / pw[len(pw) // 2], 3)}


def main():
    h, f, G, rows = 4096, 14336, 8, 1024
    g = torch.Generator(device="cuda").manual_seed(0)

    def rnd(*s):
        return (torch.randn(*s, device="cuda", generator=g) * 0.1).bfloat16()

    w1 = rnd(G, 2 * f, h); w2 = rnd(G, h, f)
    w1f, w2f, w1t = w1.reshape(G * 2 * f, h), w2.reshape(G * h, f), w1.transpose(1, 2)
    x = rnd(rows * G, h)
    grows = torch.full((G,), rows, device="cuda", dtype=torch.int32)
    offs = grows.cumsum(0).to(torch.int32)
    o1 = torch.empty(rows * G, 2 * f, device="cuda", dtype=torch.bfloat16)
    o2 = torch.empty(rows * G, f, device="cuda", dtype=torch.bfloat16)
    f1, f2 = 2.0 * rows * G * h * 2 * f, 2.0 * rows * G * h * f
    cases = [
        ("fc1_ours", lambda: ops.grouped_gemm(x, w1f, grows, N=2 * f, K=h, cta_pair=True, out=o1), f1),
        ("fc1_torch", lambda: torch._grouped_mm(x, w1t, offs=offs), f1),
        ("fc2dg_ours", lambda: ops.grouped_gemm(x, w2f, grows, N=f, K=h, b_mn_major=True, cta_pair=True, out=o2), f2),
        ("fc2dg_torch", lambda: torch._grouped_mm(x, w2, offs=offs), f2),
    ]
    res = {}
    for rnd_i, order in enumerate((cases, cases[::-1])):
        for name, fn, fl in order:
            res.setdefault(name, []).append(run(fn, fl))
            time.sleep(0.5)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
