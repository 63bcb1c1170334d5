"""Worker of test_task_halves_bit_identical: one EM step of a small ragged problem on the FP32 engine
under the CMTCS_SIMT_SPLIT setting of its environment (the library reads it once per process); prints
a SHA-256 of the posterior arrays and the step's log-likelihood and CG step count."""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import synthetic  # noqa: E402
from gpu_common import make_gpu, to_np  # noqa: E402

T, C, K, N, D = (int(a) for a in sys.argv[1:6])
data = synthetic.small_problem(T=T, C=C, N=N, D=D, K=K, sigma=0.03, seed=21, support=6)
alpha = np.random.default_rng(5).uniform(0.3, 4.0, (C, D))
m = make_gpu(data, alpha=alpha, cap=600, tol=1e-7, engine="fp32")
info = m.em_step(1)
post = to_np(m.posterior())
launches = m.kernel_launches
m.close()
h = hashlib.sha256()
for k in sorted(post):
    h.update(np.ascontiguousarray(post[k]).tobytes())
print(json.dumps({"sha": h.hexdigest(), "loglik": info["loglik"], "cg_iters": info["cg_iters"],
                  "probe_col_iters": info["probe_col_iters"], "launches": launches}))
