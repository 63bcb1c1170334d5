"""Top instructions / source lines of an ncu report by warp-stall samples.
Usage: python tools/ncu_hot.py report.ncu-rep [sass|cuda] [N]"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
view = sys.argv[2] if len(sys.argv) > 2 else "sass"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", view],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] in ("Address", "Line", "#"))
hdr = rows[hdr_i]
si = hdr.index("Warp Stall Sampling (All Samples)")


def _num(x):
    try:
        float(x or 0)
        return True
    except ValueError:
        return False


# a report with several kernels prints one table per kernel: keep the first kernel's rows
data = []
for r in rows[hdr_i + 1:]:
    if len(r) != len(hdr):
        continue
    if not _num(r[si]):
        break
    data.append(r)
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[si] or 0) for r in data)
data.sort(key=lambda r: -float(r[si] or 0))
print(f"total samples {tot:.0f}")
for r in data[:n]:
    s = float(r[si] or 0)
    top = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
    src = r[1].strip()[:90]
    print(f"{100*s/tot:5.1f}%  {r[0][-6:]:>6}  {src:90s}  " + " ".join(f"{k}:{v:.0f}" for v, k in top if v))
