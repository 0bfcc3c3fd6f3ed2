"""Per-source-line instruction / stall-sample totals of one kernel of an ncu
report, mapping the SASS page's addresses to the local build's line table.
usage: python tools/ncu_lines.py report.ncu-rep <kernel_regex> <cubin> <mangled-substring> [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kre, cubin, fname = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
# kernel_regex is matched against the mangled name (template arguments select one instantiation)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name-base",
                      "mangled", "-k", "regex:" + kre, "--launch-count", "1"], capture_output=True, text=True).stdout
lines = [ln for ln in out.splitlines() if not ln.startswith('"Kernel Name"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
R = [r for r in rows[1:] if len(r) == len(hdr) and r[0] != "Address"]
addrs = [int(r[ix["Address"]], 16) for r in R]
base = min(addrs)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
cur = None
line_of = {}
inside = False
for ln in dis.splitlines():
    if ln.startswith("//--------------------- .text."):
        inside = fname in ln
        cur = None
        continue
    if not inside:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if "//##" in ln and m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r'\s*/\*([0-9a-f]+)\*/', ln)
    if m and cur is not None:
        line_of[int(m.group(1), 16)] = cur
ins = collections.Counter()
smp = collections.Counter()
for r, a in zip(R, addrs):
    l = line_of.get(a - base, -1)
    ins[l] += int(r[ix["Instructions Executed"]] or 0)
    smp[l] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
tot_i, tot_s = sum(ins.values()), sum(smp.values())
print(f"warp instructions {tot_i}, samples {tot_s}")
for l, v in sorted(smp.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{str(l):28s} samples {100 * v / tot_s:5.1f}%  instr {100 * ins[l] / tot_i:5.1f}%")
