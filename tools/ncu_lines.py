"""Attribute an ncu report's SASS-level warp-stall samples to CUDA source lines via the cubin's line
table (nvdisasm -g).  Usage: python tools/ncu_lines.py report.ncu-rep kernel.cubin function_substring [N]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, fn = sys.argv[1:4]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# walk the function's SASS: line markers '//## File "...", line N' precede instructions '/*off*/'
line_of = {}
cur_fn = None
cur_line = None
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
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = min(int(r[0], 16) for r in data)
agg = collections.defaultdict(lambda: collections.Counter())
tot = 0.0
for r in data:
    s = float(r[si] or 0)
    tot += s
    key = line_of.get(int(r[0], 16) - base, ("?", 0))
    agg[key]["_all"] += s
    for i in stall:
        agg[key][hdr[i][6:]] += float(r[i] or 0)
src = {}
for key in agg:
    if key[0] != "?" and key[0] not in src:
        try:
            src[key[0]] = open(f"paper_2310_00420_b200/csrc/{key[0]}").read().splitlines()
        except OSError:
            src[key[0]] = []
items = sorted(agg.items(), key=lambda kv: -kv[1]["_all"])
print(f"total samples {tot:.0f}")
for (f, l), c in items[:n]:
    text = src.get(f, [])[l - 1].strip()[:70] if f in src and 0 < l <= len(src[f]) else ""
    top = sorted(((v, k) for k, v in c.items() if k != "_all"), reverse=True)[:3]
    print(f"{100 * c['_all'] / tot:5.1f}% {f}:{l:<5} {text:70s} " + " ".join(f"{k}:{v:.0f}" for v, k in top if v))
