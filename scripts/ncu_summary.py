"""Summarise ncu exports into profiles/ (tracked evidence).

  python scripts/ncu_summary.py launches <launches.csv> <out.md>
  python scripts/ncu_summary.py full <raw.csv> <out.md>
"""
import csv
import sys
from collections import OrderedDict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (elapsed)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % (active)"),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", "UTCHMMA bf16 % (elapsed)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
]
FULL_COLS = ["Kernel Name"] + [k for k, _ in KEYS]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Metric Name")
    data = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = v / 1000.0 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1000.0)
        if "moe::" not in r[ki]:
            continue
        data.append((r[ki], us))
    agg = OrderedDict()
    starts = [i for i, (n, _) in enumerate(data) if "router_logits" in n or "router_topk" in n]
    half = data[starts[-1]:] if starts else data[len(data) // 2:]   # the last step
    total = 0.0
    for name, us in half:
        short = name.replace("void ", "").split("(")[0]
        agg.setdefault(short, [0, 0.0])
        agg[short][0] += 1
        agg[short][1] += us
        total += us
    with open(out, "w") as fh:
        fh.write(f"# Kernel launch list, one fwd+bwd step (source: {path})\n\n")
        fh.write("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: "
                 "compare shares, not absolutes)\n\n| kernel | launches | us | share |\n|---|---|---|---|\n")
        for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"| `{k}` | {c} | {us:.1f} | {100 * us / total:.1f}% |\n")
        fh.write(f"| **total** | {sum(c for c, _ in agg.values())} | {total:.1f} | 100% |\n")
    print(open(out).read())


def full(path, out):
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    with open(out, "w") as fh:
        fh.write(f"# ncu --set full summary (source: {path})\n\n")
        kn = h.index("Kernel Name")
        for j, r in enumerate(rows[2:]):
            fh.write(f"## launch {j}: `{r[kn].split('(')[0]}`\n\n| metric | value | unit |\n|---|---|---|\n")
            for key, label in KEYS:
                if key in h:
                    i = h.index(key)
                    fh.write(f"| {label} (`{key}`) | {r[i]} | {u[i]} |\n")
            fh.write("\n")
    print(open(out).read())


def filter_raw(src, dst):
    rows = list(csv.reader(open(src)))
    keep = [i for i, c in enumerate(rows[0]) if c in FULL_COLS]
    with open(dst, "w") as fh:
        w = csv.writer(fh)
        for r in rows:
            w.writerow([r[i] for i in keep])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "filter":
        filter_raw(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3])
