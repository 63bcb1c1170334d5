"""One config-1 EM iteration through the C ABI with each dense engine (tensor: the persistent
tcgen05 CG kernel; fp32: the CUDA-core SGEMM loop), for compute-sanitizer (racecheck / synccheck /
memcheck, one tool per run).  Prints the step info of both."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthetic  # noqa: E402
from paper_2310_00420_b200 import CoFEM  # noqa: E402

cfg = synthetic.CONFIGS[1]
data = synthetic.generate(cfg)
for engine in ("tensor", "fp32"):
    m = CoFEM(torch.from_numpy(data["phi"]).cuda(), torch.from_numpy(data["y"]).cuda(), T=cfg.T, C=cfg.C, K=cfg.K,
              beta=cfg.beta, cg_max_iters=cfg.cg_cap, cg_rel_tol=cfg.cg_tol, probe_seed=cfg.probe_seed,
              engine=engine, learn_pi=True)
    for _ in range(2):
        info = m.em_step(1)
    torch.cuda.synchronize()
    print(engine, {k: info[k] for k in ("loglik", "cg_iters", "kernel_launches")}, "pi", m.pi())
    m.close()
print("sanitize_c1 done")
