"""T and C throughput sweeps on one GPU (the axes of the paper's
Fig. 1(e, f): CoFEM time against the number of tasks T and clusters C).

Base shape: config 3 (N = 1024, D = 4096, K = 20, σ = 0.005).  T sweep: T ∈ {8, 16, 32, 64} at C = 4
(true cluster sizes scaled from 32/16/8/8); C sweep: C ∈ {1, 2, 4, 8} model clusters at T = 64 (the
data keep their 4 true clusters).  Each point: `--warmup` EM iterations from α₀ = 1, then `--steps`
timed with CUDA events; one JSON line per point (ms per EM iteration, CG steps, active probe
column-steps, and the algorithmic fp32 TFLOP/s 4·N·D per active column-step)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthetic  # noqa: E402
from paper_2310_00420_b200 import CoFEM  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--engine", default="fp32", choices=["fp32", "tensor"])
a = ap.parse_args()
base = synthetic.CONFIGS[3]


def point(cfg, axis):
    data = synthetic.generate(cfg)
    m = CoFEM(torch.from_numpy(data["phi"]).cuda(), torch.from_numpy(data["y"]).cuda(), T=cfg.T, C=cfg.C, K=cfg.K,
              beta=cfg.beta, cg_max_iters=cfg.cg_cap, cg_rel_tol=cfg.cg_tol, probe_seed=cfg.probe_seed,
              engine=a.engine)
    for _ in range(a.warmup):
        m.em_step(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    infos = [m.em_step(1) for _ in range(a.steps)]
    e1.record()
    torch.cuda.synchronize()
    m.close()
    ms = e0.elapsed_time(e1) / a.steps
    col = sum(i["probe_col_iters"] for i in infos) / a.steps
    print(json.dumps({"axis": axis, "T": cfg.T, "C": cfg.C, "N": cfg.N, "D": cfg.D, "K": cfg.K,
                      "engine": a.engine, "em_iters_timed": f"{a.warmup}..{a.warmup + a.steps - 1}",
                      "ms_per_em_iter": ms, "ms_per_em_iter_per_task": ms / cfg.T,
                      "cg_steps": [i["cg_iters"] for i in infos], "probe_col_steps_per_em_iter": col,
                      "algorithmic_tflop_per_s": 4.0 * cfg.N * cfg.D * col / (ms * 1e-3) / 1e12}), flush=True)
    del data


t0 = time.time()
for T in (8, 16, 32, 64):
    sizes = tuple(s * T // 64 for s in base.cluster_sizes)
    point(base.replace(T=T, cluster_sizes=sizes), "T")
for C in (1, 2, 8):   # C = 4 is the T = 64 point above
    point(base.replace(C=C), "C")
print(json.dumps({"sweep_wall_s": time.time() - t0}))
