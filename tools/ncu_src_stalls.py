"""Stall / instruction summary of one kernel of an ncu report's source page.
usage: python tools/ncu_src_stalls.py report.ncu-rep <launch_index> [top_n]"""
import collections
import csv
import io
import subprocess
import sys

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
lines = [ln for ln in out.splitlines() if not ln.startswith('"Kernel Name"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
seen, R = set(), []
for r in rows[1:]:
    if len(r) != len(hdr) or r[0] == "Address" or r[0] in seen:
        continue
    seen.add(r[0])
    R.append(r)
S = lambda r: int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)   # noqa: E731
E = lambda r: int(r[ix["Instructions Executed"]] or 0)               # noqa: E731
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
print("instr", sum(map(E, R)), "samples", sum(map(S, R)))
c = collections.Counter()
for r in R:
    for s in stall_cols:
        c[s] += int(r[ix[s]] or 0)
print([(k[6:], v) for k, v in c.most_common(10)])
for r in sorted(R, key=lambda r: -S(r))[:top]:
    why = sorted(((int(r[ix[s]] or 0), s[6:]) for s in stall_cols), reverse=True)[:3]
    print(r[0][-5:], S(r), E(r), r[1].strip()[:64], [w for w in why if w[0]])
