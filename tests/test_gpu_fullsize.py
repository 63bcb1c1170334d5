"""Full-size parity: BASELINE.json configs 3-5 in bench.py's launch configuration (every task on one
GPU, the config's CG cap and tolerance, alpha0 = 1, EM iteration 0), checked against the fp64 oracle
on sampled (task, cluster) blocks — each block of Alg. 2 lines 6-9 is an
independent computation the oracle can redo one at a time — and by properties that hold at any
size (finite outputs, q rows on the simplex, alpha > 0, the Eq. 4 update from the GPU's own
posterior).  Tolerances as tests/test_gpu_parity.py; the mean systems are solved to
1e-10 on both sides (parity protocol P-mu).
"""
import numpy as np
import pytest

import synthetic
from oracle import cofem as O
from gpu_common import make_gpu, rel_inf, to_np

pytestmark = pytest.mark.gpu

MU_TOL, S_TOL, Q_TOL = 1e-4, 1e-4, 1e-3
MEAN_TOL = 1e-10


def nu_tol(nu):
    return 5e-3 + 1e-6 * np.abs(nu)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


# (config, sampled tasks, sampled clusters or None = all): C3 all clusters of 2 tasks (q checked);
# C4 (17 GB of Phi) and C5 (172,032 columns) a few blocks each, sized so the oracle takes seconds
SAMPLES = [(3, [0, 41], None), (4, [0], [0, 5]), (5, [7], [3])]


@pytest.mark.parametrize("engine", ["fp32", "tensor"])
@pytest.mark.parametrize("cid,tasks,clusters", SAMPLES)
def test_full_size_sampled_blocks(torch_cuda, cid, tasks, clusters, engine):
    """Both dense engines; the FP32 one is bench.py's default (reading E1)."""
    cfg = synthetic.CONFIGS[cid]
    data = synthetic.generate(cfg)
    g = make_gpu(data, mean_tol=MEAN_TOL, engine=engine)
    info = g.em_step(1)
    post = to_np(g.posterior())
    steps = g.transcript()["steps"].cpu().numpy().reshape(cfg.T, cfg.C, cfg.K)
    g.close()
    del data
    # properties at full size
    for k in ("mu", "s", "logdet", "q", "alpha"):
        assert np.all(np.isfinite(post[k])), k
    np.testing.assert_allclose(post["q"].sum(axis=1), 1.0, atol=1e-12)
    assert np.all(post["alpha"] > 0) and np.isfinite(info["loglik"])
    a_own = O.m_step(post["q"], post["mu"], post["s"], np.ones((cfg.C, cfg.D)))
    assert np.max(rel_inf(post["alpha"], a_own)) <= 1e-10      # Eq. 4 from the GPU's own posterior
    # sampled blocks against the oracle
    cl = list(range(cfg.C)) if clusters is None else list(clusters)
    for t in tasks:
        sub = synthetic.generate(cfg, [t])
        phi_t = sub["phi"] if cfg.shared_phi else sub["phi"][0]
        P = O.probe_signs(cfg.probe_seed, 0, cfg.T, t, cfg.C, cfg.K, cfg.D)
        o = O.cofem_task(phi_t, sub["y"][0], sub["beta"], np.ones((cfg.C, cfg.D)), sub["pi"], P, cfg.cg_tol,
                         cfg.cg_cap, mu_tol=MEAN_TOL, mu_cap=cfg.cg_cap, clusters=clusters)
        mu_err = rel_inf(post["mu"][t, cl], o["mu"])
        s_err = rel_inf(post["s"][t, cl], o["s"])
        conv = np.all(steps[t, cl] < cfg.cg_cap, axis=-1) & np.all(
            np.asarray(o["probe_steps"]).reshape(len(cl), cfg.K) < cfg.cg_cap, axis=-1)
        nu_err = np.abs(post["logdet"][t, cl] - o["nu"])
        print(f"C{cid} [{engine}] task {t} clusters {cl}: mu {mu_err.max():.2e} s {s_err.max():.2e} "
              f"nu {nu_err.max():.2e} (|nu| {np.abs(o['nu']).max():.3g}) converged {conv.sum()}/{conv.size}")
        assert mu_err.max() <= MU_TOL
        assert conv.any() and s_err[conv].max() <= S_TOL
        assert np.all(nu_err <= nu_tol(o["nu"]))
        if clusters is None:
            assert np.max(np.abs(post["q"][t] - o["q"])) <= Q_TOL
