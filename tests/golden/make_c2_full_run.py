"""Writes tests/golden/c2_full_run.json: the fp64 oracle's full 30-iteration CoFEM run of config 2
(BASELINE.json configs[1]) — final assignments, NMSE and the per-iteration log-likelihood — for the
GPU full-run parity test.  Calls only synthetic/ and oracle/ (never the CUDA path).
Run: python tests/golden/make_c2_full_run.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synthetic  # noqa: E402
from oracle import cofem as O  # noqa: E402


def main():
    cfg = synthetic.CONFIGS[2]
    data = synthetic.generate(cfg)
    caps = []
    orc = O.run(data, cfg.em_iters,
                callback=lambda i, e, a: caps.append(int(np.sum(e["probe_steps"] >= cfg.cg_cap))))
    out = {"config": cfg.name, "em_iters": cfg.em_iters, "assign": [int(a) for a in orc["assign"]],
           "nmse": float(orc["nmse"]), "L": [float(h["L"]) for h in orc["history"]],
           "probe_cap_hits": caps,
           "source": "oracle.cofem.run(synthetic.generate(CONFIGS[2]), 30), alpha0 = 1, fp64 (this script)"}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c2_full_run.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(out["assign"], out["nmse"])


if __name__ == "__main__":
    main()
