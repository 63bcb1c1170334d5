"""Run `--warmup` EM iterations of a config, then ONE EM iteration inside cudaProfilerStart/Stop
(for `ncu --profile-from-start off ...`).  Prints the step info and the library's event timing."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic  # noqa: E402
from paper_2310_00420_b200 import CoFEM  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2, help="1-6 (6: partial Fourier)")
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--tasks", type=int, default=0, help="use only the first n tasks (0 = all)")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--engine", default="tensor", choices=["tensor", "fp32"])
a = ap.parse_args()
cfg = synthetic.CONFIGS[a.config]
tasks = range(a.tasks) if a.tasks else None
data = synthetic.generate(cfg, tasks)
if cfg.operator == "fourier":   # config 6: Φ_t = Ω_t F given by its sampled rows
    m = CoFEM(None, torch.from_numpy(data["y"]).cuda(), fourier_rows=torch.from_numpy(data["rows"]).cuda(), D=cfg.D,
              T=cfg.T, C=cfg.C, K=cfg.K, beta=cfg.beta, cg_max_iters=cfg.cg_cap, cg_rel_tol=cfg.cg_tol,
              probe_seed=cfg.probe_seed)
else:
    m = CoFEM(torch.from_numpy(data["phi"]).cuda(), torch.from_numpy(data["y"]).cuda(), T=cfg.T, C=cfg.C, K=cfg.K,
              beta=cfg.beta, cg_max_iters=cfg.cg_cap, cg_rel_tol=cfg.cg_tol, probe_seed=cfg.probe_seed,
              shared_phi=cfg.shared_phi, engine=a.engine)
for _ in range(a.warmup):
    m.em_step(1)
m.set_timing(True)
torch.cuda.synchronize()
torch.cuda.profiler.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    info = m.em_step(1)
e1.record()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ms = e0.elapsed_time(e1) / a.steps
print(json.dumps({"em_ms": ms, "us_per_cg_step": 1e3 * ms / max(1, info["cg_iters"]), "info": info,
                  "timing": m.get_timing()}))
