"""Parity of the partial-Fourier path (the paper's own sensing matrix
Φ_t = Ω_t F) with the fp64 oracle, which applies the DENSE real-embedded partial DFT
(oracle.cofem.partial_fourier_matrix, pinned in tests/test_oracle_pins.py against numpy's FFT,
Parseval and the circulant spectrum).  The GPU applies ΦᵀΦ by FFT inside k_cg_fourier (one CTA per
column, vectors on chip).  Bars as tests/test_gpu_parity.py: the mean systems in fp64
on both sides to 1e-10; probe columns fp32 (FFT error ~log₂D·ε₃₂) with fp64 dots.
"""
import numpy as np
import pytest

import synthetic
from oracle import cofem as O
from gpu_common import compare_step, make_gpu, rel_inf, to_np

pytestmark = pytest.mark.gpu

MU_TOL, S_TOL, Q_TOL, A_TOL, L_TOL = 1e-4, 1e-4, 1e-3, 1e-4, 1e-3
MEAN_TOL = 1e-10


def nu_tol(nu):
    return 5e-3 + 1e-6 * np.abs(nu)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def small_fourier(T=3, C=2, D=512, N=128, K=6, sigma=0.05, seed=41, support=20):
    cfg = synthetic.CONFIGS[6].replace(cfg_id=140 + seed, T=T, C=C, D=D, N=N, K=K, sigma=sigma,
                                       cluster_sizes=tuple([T // C + (1 if j < T % C else 0) for j in range(C)]),
                                       support=support, cg_cap=4 * D)
    return synthetic.generate(cfg)


@pytest.mark.parametrize("C,K,D", [(2, 6, 512), (3, 5, 1024)])
def test_fourier_rhs_and_operator_through_one_step(torch_cuda, C, K, D):
    """A single EM step on a small partial-Fourier problem from an asymmetric state: μ, s, ν̄, q, L
    and α against the oracle (dense DFT Φ), every block converged on both sides.  (3, 5): an odd
    number of probe columns per task — the paired-column kernel's last pair has one column — and
    an even log₂D (the FFT's radix-4 passes without the closing radix-2 stage)."""
    data = small_fourier(C=C, K=K, T=3, D=D, N=D // 4)
    cfg = data["cfg"]
    alpha = np.random.default_rng(3).uniform(0.5, 5.0, (cfg.C, cfg.D))
    g = make_gpu(data, alpha=alpha, em_iter0=2, cap=cfg.cg_cap, tol=1e-7, mean_tol=MEAN_TOL)
    info = g.em_step(1)
    post = to_np(g.posterior())
    steps = g.transcript()["steps"].cpu().numpy().reshape(cfg.T, cfg.C, cfg.K)
    g.close()
    orc = O.e_step(data, alpha, 2, tol=1e-7, cap=cfg.cg_cap, mu_tol=MEAN_TOL, mu_cap=cfg.cg_cap)
    a_next = O.m_step(orc["q"], orc["mu"], orc["s"], alpha)
    conv = np.all(steps < cfg.cg_cap, axis=-1) & np.all(orc["probe_steps"].reshape(steps.shape) < cfg.cg_cap, axis=-1)
    e = compare_step(post, info, orc, a_next, conv)
    print("fourier small", e, "converged", conv.sum(), "/", conv.size, "GPU steps", steps.max())
    assert e["mu"] <= MU_TOL
    assert conv.all() and e["s_conv"] <= S_TOL
    assert np.all(np.abs(post["logdet"] - orc["nu"]) <= nu_tol(orc["nu"]))
    assert e["q_abs"] <= Q_TOL and e["L_abs"] <= L_TOL
    if np.max(np.abs(post["q"] - orc["q"])) <= 1e-5:
        assert e["alpha"] <= A_TOL


def test_fourier_prior_only_closed_form(torch_cuda):
    """No sampled rows would be Φ = 0; with β → tiny the operator is diag(α): s = 1/α and
    ν̄ = −Σ log α, here with a near-zero β so the closed form holds to rounding."""
    data = small_fourier(T=2, C=2, seed=42)
    data["beta"] = 1e-12
    alpha = np.stack([np.repeat([0.5, 2.0], 256), np.repeat([1.5, 4.0], 256)])
    g = make_gpu(data, alpha=alpha, cap=50, tol=1e-12)
    g.em_step(1)
    post = to_np(g.posterior())
    g.close()
    np.testing.assert_allclose(post["s"], np.broadcast_to(1.0 / alpha, post["s"].shape), rtol=1e-5)
    np.testing.assert_allclose(post["logdet"], np.broadcast_to(-np.log(alpha).sum(1), (2, 2)), rtol=1e-5, atol=1e-3)


def test_fourier_config6_sampled_blocks(torch_cuda):
    """The paper's workload at full size (config 6: D = 8192, N = 2048 sampled rows, 64 tasks, C = 4,
    K = 15, the paper's cap U = 50) in the launch configuration bench.py times, EM iteration 0 from
    α₀ = 1: sampled tasks against the oracle (dense 4096 × 8192 Φ_t per task), all clusters of each
    (q checked); properties of every output at full size."""
    cfg = synthetic.CONFIGS[6]
    data = synthetic.generate(cfg)
    g = make_gpu(data, mean_tol=MEAN_TOL)
    info = g.em_step(1)
    post = to_np(g.posterior())
    steps = g.transcript()["steps"].cpu().numpy().reshape(cfg.T, cfg.C, cfg.K)
    g.close()
    for k in ("mu", "s", "logdet", "q", "alpha"):
        assert np.all(np.isfinite(post[k])), k
    np.testing.assert_allclose(post["q"].sum(axis=1), 1.0, atol=1e-12)
    for t in (0, 37):
        sub = synthetic.generate(cfg, [t])
        o = O.e_step(sub, np.ones((cfg.C, cfg.D)), 0, mu_tol=MEAN_TOL, mu_cap=cfg.cg_cap)
        mu_e = rel_inf(post["mu"][t], o["mu"][0])
        s_e = rel_inf(post["s"][t], o["s"][0])
        conv = np.all(steps[t] < cfg.cg_cap, axis=-1) & np.all(o["probe_steps"][0].reshape(cfg.C, cfg.K) < cfg.cg_cap, axis=-1)
        nu_e = np.abs(post["logdet"][t] - o["nu"][0])
        print(f"C6 task {t}: mu {mu_e.max():.2e} s {s_e.max():.2e} nu {nu_e.max():.2e} q "
              f"{np.max(np.abs(post['q'][t] - o['q'][0])):.2e} converged {conv.sum()}/{conv.size}")
        assert mu_e.max() <= MU_TOL
        assert conv.any() and s_e[conv].max() <= S_TOL
        assert np.all(nu_e <= nu_tol(o["nu"][0]))
        assert np.max(np.abs(post["q"][t] - o["q"][0])) <= Q_TOL
