"""Summarise an `ncu --set full` report: per kernel launch duration, DRAM bytes, L2 bytes, tensor /
FMA pipe activity, top stall reasons.  Usage: python tools/ncu_summary.py report.ncu-rep > out.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "lts_bytes": "lts__t_bytes.sum",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "grid_size": "launch__grid_size",
    "registers": "launch__registers_per_thread",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
         "ns": 1, "us": 1e3, "ms": 1e6}


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        k = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]}
        for name, key in KEYS.items():
            if key in hdr:
                i = hdr.index(key)
                try:
                    k[name] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    k[name] = r[i]
        tensor = [h for h in hdr if h.startswith("sm__pipe_tensor") and h.endswith("pct_of_peak_sustained_active")]
        for h in tensor:
            try:
                k[h] = float(r[hdr.index(h)])
            except ValueError:
                pass
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        k["top_stalls"] = {n: v for v, n in sorted(stalls, reverse=True)[:6]}
        out.append(k)
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
