"""The library's NCCL path (ncclCommInitRank + the per-EM-iteration ncclAllReduce of the Eq. 4
sums, csrc/cmtcs_api.cu) on >= 2 GPUs: a sharded run equals a single-context run.  Skipped on a
1-GPU box (the shard algebra itself is covered there by test_task_shards_match_whole, which
compares each shard context's pre-all-reduce sums, cmtcs_estep_sums, with the whole problem's)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_nccl_allreduce_sharded_run_matches_single_context():
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(HERE, "nccl_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0


def test_nccl_path_single_rank_matches_no_communicator():
    """The library's NCCL plumbing on one GPU: a context given an NCCL unique id with world = 1
    creates a 1-rank communicator (ncclCommInitRank) and runs the Eq. 4 all-reduce through
    ncclAllReduce on its stream every EM iteration; the run must equal the communicator-free run
    bit for bit (a 1-rank sum is a copy) — config 2, 3 EM iterations, both dense engines."""
    import numpy as np
    import torch
    sys.path.insert(0, HERE)
    import synthetic
    from gpu_common import to_np
    from paper_2310_00420_b200 import CoFEM, cmtcs
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    cfg = synthetic.CONFIGS[2]
    data = synthetic.generate(cfg)
    for engine in ("fp32", "tensor"):
        runs = []
        for uid in (None, cmtcs.cmtcs_get_unique_id()):
            phi = torch.from_numpy(data["phi"]).cuda()
            y = torch.from_numpy(data["y"]).cuda()
            m = CoFEM(phi, y, T=cfg.T, C=cfg.C, K=cfg.K, beta=cfg.beta, cg_max_iters=cfg.cg_cap,
                      cg_rel_tol=cfg.cg_tol, probe_seed=cfg.probe_seed, pi=data["pi"], alpha0=data["alpha0"],
                      engine=engine, nccl_uid=uid, rank=0, world=1)
            L = [m.em_step(1)["loglik"] for _ in range(3)]
            runs.append((L, to_np(m.posterior())))
            m.close()
        (L0, p0), (L1, p1) = runs
        assert L0 == L1, (engine, L0, L1)
        for k in ("alpha", "q", "mu"):
            np.testing.assert_array_equal(p0[k], p1[k], err_msg=f"{engine} {k}")
