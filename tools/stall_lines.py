"""Per-source-line warp-stall attribution of an ncu capture (SASS page) using nvdisasm line info.

  python tools/stall_lines.py report.ncu-rep kernel.cubin <mangled-kernel-prefix> [top]
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, cubin, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.check_output(["nvdisasm", "--print-line-info", cubin], text=True)
cur, on, a2l = None, False, {}
for l in dis.split("\n"):
    if l.startswith("\t.section\t.text.") or l.startswith(".section\t.text."):
        on = fn in l
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if on and m and cur:
        a2l.setdefault(int(m.group(1), 16), cur)
src = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], text=True)
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
R = rows[2:]
# a capture of several launches repeats the header per launch: keep the first launch's rows
for k, r in enumerate(R):
    if "Address" in r or "Kernel Name" in r:
        R = R[:k]
        break
ix = {h: i for i, h in enumerate(hdr)}
base = int(R[0][ix["Address"]], 16)
S = "Warp Stall Sampling (All Samples)"
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot, ex, agg = defaultdict(int), defaultdict(int), defaultdict(lambda: defaultdict(int))
for r in R:
    ln = a2l.get(int(r[ix["Address"]], 16) - base, ("?", 0))
    tot[ln] += int(r[ix[S]] or 0)
    ex[ln] += int(r[ix["Instructions Executed"]] or 0)
    for s in stalls:
        agg[ln][s] += int(r[ix[s]] or 0)
T = sum(tot.values())
E = sum(ex.values())
print(f"samples {T}  warp instructions {E}")
import os
key = ex if os.environ.get("SORT") == "exec" else tot
for ln, v in sorted(key.items(), key=lambda x: -x[1])[:top]:
    v = tot[ln]
    st = dict(sorted(((k.replace("stall_", ""), c) for k, c in agg[ln].items() if c), key=lambda x: -x[1])[:4])
    print(f"{ln[0]}:{ln[1]:<5} {v:6d} {100 * v / T:5.1f}%  exec {ex[ln]:9d} {st}")
