#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run in the build container).

    python tools/ncu_summary.py launches <launches.csv>      # per-kernel shares
    python tools/ncu_summary.py full <report.ncu-rep>         # key metrics per launch

The launch list comes from `ncu --metrics gpu__time_duration.sum
--clock-control none --csv` (cold-cache, serialised: compare shares, not
absolutes); the full report from `ncu --set full`.
"""

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "time_us"),
    ("dram__bytes_read.sum", "dram_read_MB"),
    ("dram__bytes_write.sum", "dram_write_MB"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pct"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    return name.split("(")[0][:90]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        us = v / 1000.0 if unit in ("nsecond", "ns") else (v * 1000.0 if unit in ("msecond", "ms") else v)
        k = short(d["Kernel Name"])
        if "gbuffer_kernel" in k or "shadowmap_kernel" in k or "spin_kernel" in k:
            continue                      # input producers (untimed setup); bench's profiling spin
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total µs | share |", "|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f} % |")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = ["| kernel | " + " | ".join(k for _, k in KEYS) + " |",
           "|---|" + "---|" * len(KEYS)]
    recs = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": short(d.get("Kernel Name", "?"))}
        cells = []
        for m, k in KEYS:
            v = d.get(m, "")
            u = units[hdr.index(m)] if m in hdr else ""
            try:
                x = float(v.replace(",", ""))
                if m.startswith("dram__bytes"):
                    x = x * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)   # -> MB
                if m == "gpu__time_duration.sum":
                    x = x * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                             "ms": 1e3}.get(u, 1.0)   # -> us
                rec[k] = x
                cells.append(f"{x:.3g}")
            except ValueError:
                cells.append(v)
        recs.append(rec)
        out.append(f"| `{rec['kernel']}` | " + " | ".join(cells) + " |")
    return "\n".join(out), recs


KMAP = {"enc0_kernel": "enc0_fused", "dec0p_kernel": "dec0_fused", "dec0_ring_kernel": "dec0_ring",
        "recon_kernel": "recon", "feat5_kernel": "feat5_blocker", "enc0_s2d_kernel": "enc0_s2d"}


def traffic(path, frames_per_launch, out, source, workload="cfg4-1080p-soft-window8"):
    """profiles/traffic.json for bench.py's roofline.traffic: DRAM bytes per
    frame of each kernel's first launch in a --set full report."""
    _, recs = full(path)
    import os
    res = json.load(open(out)) if os.path.exists(out) else {}
    res = {k: v for k, v in res.items() if v.get("workload") != workload}   # replace this workload's rows
    seen = set()
    for r in recs:
        for k, name in KMAP.items():
            if k in r["kernel"] and name not in seen and "dram_read_MB" in r:
                seen.add(name)
                res[name if workload == "cfg4-1080p-soft-window8" else f"{name}@{workload}"] = {"dram_bytes_per_frame": (r["dram_read_MB"] + r["dram_write_MB"]) * 1e6 /
                             frames_per_launch, "source": source, "workload": workload}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "traffic":      # traffic <report> <frames_per_launch> <out.json> <source-label> [workload]
        traffic(path, int(sys.argv[3]), sys.argv[4], sys.argv[5], *sys.argv[6:7])
    elif mode == "launches":
        print(launches(path))
    else:
        table, recs = full(path)
        print(table)
        if len(sys.argv) > 3:
            json.dump(recs, open(sys.argv[3], "w"), indent=1)
