"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[start + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0].split("::")[-1]
            agg[name].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3))
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k:28s} n={len(v):5d} total={sum(v):11.1f}us mean={sum(v) / len(v):9.2f}us share={sum(v) / tot:.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
