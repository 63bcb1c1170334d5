"""Per-source-line instruction counts and warp-stall samples of an ncu report (SASS rows mapped to
lines via the cubin's line table).  Usage:
  python tools/ncu_linestats.py report.ncu-rep kernel.cubin function_substring first_line last_line"""
import collections
import csv
import re
import subprocess
import sys

rep, cubin, fn, l0, l1 = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
line_of, cur_fn, cur_line = {}, None, None
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1)
        continue
    if cur_fn is None or fn not in cur_fn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur_line = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_line:
        line_of[int(m.group(1), 16)] = cur_line
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
ai, si, ie = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter()])
base = None
for r in rows[hi + 1:]:
    if len(r) != len(hdr):
        continue
    a = int(r[ai], 16)
    if base is None:
        base = a
    key = line_of.get(a - base)
    if not key or not (l0 <= key[1] <= l1):
        continue
    g = agg[key]
    g[0] += float(r[ie] or 0)
    g[1] += float(r[si] or 0)
    for i in st:
        g[2][hdr[i][6:]] += float(r[i] or 0)
src = {}
for k in agg:
    pass
for key in sorted(agg):
    ins, smp, c = agg[key]
    top = " ".join(f"{k}:{int(v)}" for k, v in c.most_common(3) if v)
    print(f"{key[0]}:{key[1]:5d}  inst {ins:12.0f}  samples {smp:8.0f}  {top}")
