"""Summarise warp-stall samples of an ncu report's source page by SASS
region: python tools/ncu_stalls.py report.ncu-rep [top_n] [kernel_regex]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kfilt = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-count", "1"] + kfilt, capture_output=True, text=True).stdout
lines = [ln for ln in out.splitlines() if not ln.startswith('"Kernel Name"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
hdr = rows[0]
rows = [r for r in rows[1:] if len(r) == len(hdr) and r[0] != "Address"]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for r in rows:
    for h in stall_cols:
        tot[h] += int(r[ix[h]] or 0)
allsamp = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in rows)
print("total samples", allsamp)
for h, v in tot.most_common():
    if v:
        print(f"  {h:24s} {v:8d} {100 * v / max(allsamp, 1):5.1f}%")
print(f"\ntop {top} instructions by samples:")
rs = sorted(rows, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:top]
for r in rs:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    why = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stall_cols), reverse=True)[:3]
    print(f"{r[0][-5:]} {s:6d} {r[1].strip()[:60]:60s} " + " ".join(f"{n}:{v}" for v, n in why if v))
