"""Pins for the CPU oracle (oracle/cofem.py) against what the paper and the mathematics fix.

Nothing here re-types an oracle formula: expected values come from closed forms, worked examples
(tests/golden/, each cited), invariants, independent library routines (LAPACK Cholesky/eigh,
scipy logm, scipy multivariate_normal) or brute force on tiny inputs.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg
import scipy.stats

import synthetic
from oracle import cofem as O


def rand_spd(D, rng, cond=50.0):
    Q, _ = np.linalg.qr(rng.standard_normal((D, D)))
    lam = np.exp(rng.uniform(0, math.log(cond), D))
    return (Q * lam) @ Q.T


def dense_cg(A, b, tol, cap):
    return O.conjugate_gradient(lambda V, cols: A @ V, b[:, None], tol, cap)


# ---------------------------------------------------------------- probes (A6) -------------
def test_splitmix64_published_vectors(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "splitmix64.json")))
    w = np.arange(len(g["outputs_hex"]), dtype=np.uint64)
    got = O.probe_word(g["seed"], w)
    assert [f"{int(x):016x}" for x in got] == g["outputs_hex"]


def test_probe_signs_values_and_balance():
    P = O.probe_signs(12345, 3, 10, 7, 4, 50, 130)
    assert P.shape == (4, 50, 130)
    assert set(np.unique(P)) == {-1.0, 1.0}
    assert abs(P.mean()) < 0.05                       # 26,000 fair signs: 5σ ≈ 0.031
    # distinct (it, t, c, k) give distinct streams
    assert not np.array_equal(P[0, 0], P[0, 1]) and not np.array_equal(P[0, 0], P[1, 0])
    Q = O.probe_signs(12345, 4, 10, 7, 4, 50, 130)
    assert np.mean(P == Q) < 0.6


def test_probe_bit_layout_brute_force():
    """Bit (d mod 64) of word w (LSB = bit 0) decides p_d; w counts 64-entry chunks (A6)."""
    seed, it, T, t, C, K, D = 99, 2, 5, 3, 2, 3, 70
    P = O.probe_signs(seed, it, T, t, C, K, D)
    M = (1 << 64) - 1
    for c in range(C):
        for k in range(K):
            for d in (0, 1, 63, 64, 69):
                w = ((((it * T + t) * C + c) * K + k) * 2) + d // 64
                z = (seed + (w + 1) * 0x9E3779B97F4A7C15) & M
                z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
                z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
                z ^= z >> 31
                assert P[c, k, d] == (1.0 if ((z >> (d % 64)) & 1) == 0 else -1.0)


# ---------------------------------------------------------------- Alg. 1 -----------------
def test_cg_scaled_identity_one_step():
    r = dense_cg(2.0 * np.eye(2), np.array([6.0, 8.0]), 1e-12, 5)
    assert r["steps"][0] == 1
    np.testing.assert_allclose(r["x"][:, 0], [3.0, 4.0], rtol=0, atol=1e-14)
    assert r["gamma"][0, 0] == pytest.approx(0.5, abs=1e-15)


def test_cg_two_distinct_eigenvalues_two_steps():
    r = dense_cg(np.diag([1.0, 4.0]), np.array([1.0, 1.0]), 1e-12, 10)
    assert r["steps"][0] == 2
    np.testing.assert_allclose(r["x"][:, 0], [1.0, 0.25], atol=1e-14)


def test_cg_matches_cholesky_solve():
    rng = np.random.default_rng(1)
    A = rand_spd(32, rng, cond=100.0)
    b = rng.standard_normal(32)
    r = dense_cg(A, b, 1e-13, 400)
    x = scipy.linalg.cho_solve(scipy.linalg.cho_factor(A), b)
    np.testing.assert_allclose(r["x"][:, 0], x, rtol=1e-9, atol=1e-11)
    assert r["relres"][0] <= 1e-13


def test_cg_error_A_norm_monotone_not_residual():
    """The A-norm of the error is non-increasing (CG theory); the residual norm need not be."""
    rng = np.random.default_rng(2)
    grew = 0
    for trial in range(20):
        A = rand_spd(24, rng, cond=1e5)
        b = rng.standard_normal(24)
        xs = scipy.linalg.solve(A, b, assume_a="pos")
        errs, ress = [], []
        for U in range(1, 25):
            x = dense_cg(A, b, 0.0, U)["x"][:, 0]
            e = x - xs
            errs.append(e @ A @ e)
            ress.append(np.linalg.norm(b - A @ x))
        assert all(errs[i + 1] <= errs[i] * (1 + 1e-9) + 1e-20 for i in range(len(errs) - 1))
        grew += sum(ress[i + 1] > ress[i] for i in range(len(ress) - 1))
    assert grew > 0          # SPEC.md:148's "residual monotone" claim is false


def test_cg_columns_independent_and_zero_rhs():
    rng = np.random.default_rng(3)
    A = rand_spd(16, rng)
    B = rng.standard_normal((16, 4))
    B[:, 2] = 0.0
    r = O.conjugate_gradient(lambda V, cols: A @ V, B, 1e-8, 40)
    assert r["steps"][2] == 0 and np.all(r["x"][:, 2] == 0)
    for j in (0, 1, 3):
        rj = O.conjugate_gradient(lambda V, cols: A @ V, B[:, j:j + 1], 1e-8, 40)
        assert rj["steps"][0] == r["steps"][j]
        np.testing.assert_allclose(rj["x"][:, 0], r["x"][:, j], rtol=1e-10, atol=1e-12)


def test_cg_breakdown_on_indefinite():
    with pytest.raises(O.Breakdown):
        dense_cg(np.diag([1.0, -1.0]), np.array([0.0, 1.0]), 1e-10, 5)


def test_cg_first_residual_is_b_and_stops_at_cap():
    rng = np.random.default_rng(4)
    A = rand_spd(20, rng, cond=1e4)
    b = rng.standard_normal(20)
    r = dense_cg(A, b, 0.0, 3)
    assert r["steps"][0] == 3
    assert r["gamma"][0, 0] == pytest.approx((b @ b) / (b @ A @ b), rel=1e-14)


# ---------------------------------------------------------------- Eq. 7-9 ----------------
def test_eq7_worked_examples(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "eq7_tridiagonal.json")))
    for c in g["cases"]:
        np.testing.assert_allclose(O.assemble_tridiagonal(np.array(c["gamma"]), np.array(c["xi"])),
                                   np.array(c["Gamma"]), rtol=1e-15, atol=1e-15)


def test_eq7_lanczos_eigenvalues_equal_A_at_full_steps():
    """Γ̄ from D steps of CG is the Lanczos tridiagonalisation of A: same spectrum."""
    rng = np.random.default_rng(5)
    Q, _ = np.linalg.qr(rng.standard_normal((12, 12)))
    lam = np.linspace(1.0, 4.0, 12)                      # well separated: no Lanczos ghosts
    A = (Q * lam) @ Q.T
    p = np.where(rng.random(12) < 0.5, -1.0, 1.0)
    r = dense_cg(A, p, 0.0, 12)
    G = O.assemble_tridiagonal(r["gamma"][:, 0], r["xi"][:, 0])
    np.testing.assert_allclose(np.linalg.eigvalsh(G), lam, rtol=1e-8)


def test_eq7_logdet_identity_and_unit_first_row():
    """Γ̄ = Bᵀdiag(1/γ)B with B unit bidiagonal ⇒ Σ log λ̄ = −Σ log γ; and Σ_u S̄²_{u,1} = 1."""
    rng = np.random.default_rng(6)
    gam = rng.uniform(0.1, 3.0, 40)
    xi = rng.uniform(0.01, 2.0, 39)
    G = O.assemble_tridiagonal(gam, xi)
    lam, V = np.linalg.eigh(G)
    assert np.sum(np.log(lam)) == pytest.approx(-np.sum(np.log(gam)), rel=1e-12)
    assert np.sum(V[0] ** 2) == pytest.approx(1.0, abs=1e-12)


def test_eq8_quadrature_exact_at_U_equals_D():
    """with U = D steps, D·Σ S²_{u,1} log λ_u = pᵀ log(A) p (scipy logm)."""
    rng = np.random.default_rng(7)
    for trial in range(3):
        A = rand_spd(16, rng, cond=30.0)
        p = np.where(rng.random(16) < 0.5, -1.0, 1.0)
        r = dense_cg(A, p, 0.0, 16)
        tau = O.quadrature_term(r["gamma"][:, 0], r["xi"][:, 0], 16)
        want = p @ np.real(scipy.linalg.logm(A)) @ p
        assert tau == pytest.approx(want, rel=1e-8)


def test_eq9_scaled_identity_exact():
    """A = cI: one CG step, ν̄ = −D log c exactly for any K."""
    D, c = 10, 2.0
    terms = []
    rng = np.random.default_rng(8)
    for k in range(5):
        p = np.where(rng.random(D) < 0.5, -1.0, 1.0)
        r = dense_cg(c * np.eye(D), p, 1e-12, 10)
        assert r["steps"][0] == 1
        terms.append(O.quadrature_term(r["gamma"][:1, 0], r["xi"][:1, 0], D))
    assert O.estimate_logdet(np.array(terms)) == pytest.approx(-D * math.log(c), rel=1e-14)


def test_prior_only_task_is_exact():
    """Φ = 0: A = diag(α) ⇒ s = 1/α and ν̄ = −Σ log α exactly, μ = 0."""
    D, N, C, K = 12, 5, 2, 3
    rng = np.random.default_rng(9)
    alpha = np.stack([rng.choice([0.5, 2.0, 7.0], D), rng.choice([1.5, 3.0], D)])
    P = np.where(rng.random((C, K, D)) < 0.5, -1.0, 1.0)
    r = O.cofem_task(np.zeros((N, D)), rng.standard_normal(N), 3.0, alpha, np.full(C, 0.5), P,
                     1e-13, 50)
    np.testing.assert_allclose(r["s"], 1.0 / alpha, rtol=1e-12)
    np.testing.assert_allclose(r["nu"], -np.log(alpha).sum(1), rtol=1e-12)
    np.testing.assert_allclose(r["mu"], 0.0, atol=1e-15)


# ---------------------------------------------------------------- Eq. 5 ------------------
def test_eq5_identity_and_diagonal_closed_forms():
    rng = np.random.default_rng(10)
    P = np.where(rng.random((7, 9)) < 0.5, -1.0, 1.0)
    np.testing.assert_array_equal(O.estimate_diagonal(P, P), np.ones(9))         # Σ = I
    dg = rng.uniform(0.5, 3, 9)
    np.testing.assert_allclose(O.estimate_diagonal(P, P * dg), dg, rtol=1e-15)   # diagonal Σ


def test_eq5_unbiased_monte_carlo():
    rng = np.random.default_rng(11)
    A = rand_spd(20, rng, cond=10.0)
    S = np.linalg.inv(A)
    K = 4000
    P = np.where(rng.random((K, 20)) < 0.5, -1.0, 1.0)
    X = P @ S
    s = O.estimate_diagonal(P, X)
    se = np.std(P * X, axis=0) / math.sqrt(K)
    assert np.all(np.abs(s - np.diag(S)) <= 5 * se + 1e-12)


# ---------------------------------------------------------------- Eq. 3 ------------------
def test_softmax_worked_examples(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "softmax_responsibilities.json")))
    for c in g["cases"]:
        np.testing.assert_allclose(O.responsibilities(np.array(c["ell"]), np.array(c["pi"])), c["q"],
                                   rtol=1e-14)
    e = np.array([1.0, -2.0, 5.0])
    np.testing.assert_allclose(O.responsibilities(e, np.full(3, 1 / 3)),
                               O.responsibilities(e + 1234.5, np.full(3, 1 / 3)), rtol=1e-12)
    with pytest.raises(ArithmeticError):
        O.responsibilities(np.array([-np.inf, -np.inf]), np.array([0.5, 0.5]))


def test_ell_is_gaussian_evidence():
    """½ℓ̃ + (N/2)log(β/2π) = log N(y; 0, β⁻¹I + Φ diag(α)⁻¹Φᵀ) with exact μ and log det Σ,
    and the literal PAPER.md:59 form differs from ℓ̃ by exactly β‖y‖² (reading A1)."""
    rng = np.random.default_rng(12)
    N, D, beta = 8, 16, 7.0
    phi = rng.standard_normal((N, D)) / math.sqrt(N)
    y = rng.standard_normal(N)
    alpha = rng.uniform(0.2, 5.0, (1, D))
    e = O.exact_task(phi, y, beta, alpha, np.ones(1))
    cov = np.eye(N) / beta + phi @ np.diag(1 / alpha[0]) @ phi.T
    want = scipy.stats.multivariate_normal(np.zeros(N), cov).logpdf(y)
    assert 0.5 * e["ell"][0] + 0.5 * N * math.log(beta / (2 * math.pi)) == pytest.approx(want, rel=1e-12)
    assert e["ll"] == pytest.approx(want, rel=1e-12)
    lit = O.ell_literal(e["nu"][0], alpha[0], beta, y, phi @ e["mu"][0])
    assert lit - e["ell"][0] == pytest.approx(beta * y @ y, rel=1e-10)


def test_exact_estep_against_lapack():
    rng = np.random.default_rng(13)
    N, D, beta = 6, 10, 4.0
    phi = rng.standard_normal((N, D))
    y = rng.standard_normal(N)
    alpha = rng.uniform(0.5, 2.0, (2, D))
    e = O.exact_task(phi, y, beta, alpha, np.array([0.3, 0.7]))
    for c in range(2):
        A = beta * phi.T @ phi + np.diag(alpha[c])
        S = scipy.linalg.inv(A)
        np.testing.assert_allclose(e["mu"][c], beta * S @ phi.T @ y, rtol=1e-10)
        np.testing.assert_allclose(e["s"][c], np.diag(S), rtol=1e-10)
        assert e["nu"][c] == pytest.approx(-np.linalg.slogdet(A)[1], rel=1e-12)
    assert e["q"].sum() == pytest.approx(1.0, abs=1e-14)


# ---------------------------------------------------------------- Eq. 4 ------------------
def test_mstep_closed_forms():
    a = O.m_step(np.ones((1, 1)), np.ones((1, 1, 3)), np.ones((1, 1, 3)), np.ones((1, 3)))
    np.testing.assert_allclose(a, 0.5)
    a = O.m_step(np.ones((1, 1)), np.zeros((1, 1, 2)), np.zeros((1, 1, 2)), np.ones((1, 2)),
                 alpha_max=1e12)
    np.testing.assert_allclose(a, 1e12)                                  # divergence → cap
    old = np.array([[3.0, 4.0], [5.0, 6.0]])
    q = np.array([[1.0, 0.0], [1.0, 0.0]])
    a = O.m_step(q, np.ones((2, 2, 2)), np.ones((2, 2, 2)), old)
    np.testing.assert_array_equal(a[1], old[1])                          # empty cluster keeps α
    np.testing.assert_allclose(a[0], 0.5)


def test_mstep_single_cluster_is_multitask_cs():
    """C = 1: α_d = T / Σ_t (μ_td² + s_td) (multi-task CS update)."""
    rng = np.random.default_rng(14)
    T, D = 5, 7
    mu = rng.standard_normal((T, 1, D))
    s = rng.uniform(0.1, 1.0, (T, 1, D))
    a = O.m_step(np.ones((T, 1)), mu, s, np.ones((1, D)))
    np.testing.assert_allclose(a[0], T / np.sum(mu[:, 0] ** 2 + s[:, 0], axis=0), rtol=1e-14)


def test_mstep_sharded_sums_equal_whole():
    rng = np.random.default_rng(15)
    q = rng.dirichlet(np.ones(3), size=9)
    mu = rng.standard_normal((9, 3, 5))
    s = rng.uniform(-0.1, 1.0, (9, 3, 5))
    n1, d1 = O.m_step_sums(q[:4], mu[:4], s[:4])
    n2, d2 = O.m_step_sums(q[4:], mu[4:], s[4:])
    np.testing.assert_allclose(O.m_step_finish(n1 + n2, d1 + d2, np.ones((3, 5))),
                               O.m_step(q, mu, s, np.ones((3, 5))), rtol=1e-13)


# ---------------------------------------------------------------- EM as a whole ----------
def test_exact_em_likelihood_monotone():
    """EM theory: L(θ̃) ≥ L(θ̂) in exact mode (asymmetric α₀, A4)."""
    data = synthetic.small_problem(T=4, C=2, N=12, D=24, sigma=0.1, seed=3, support=3)
    rng = np.random.default_rng(0)
    alpha0 = rng.uniform(0.0, 1.0, (2, 24)) + 1e-3        # Alg. 2 line 1: Uniform(0,1)
    r = O.run(data, 25, mode="exact", alpha0=alpha0)
    L = [h["L"] for h in r["history"]]
    assert all(L[i + 1] >= L[i] - 1e-9 * abs(L[i]) for i in range(len(L) - 1))
    assert L[-1] > L[0]


def test_mstep_pi_maximises_the_surrogate_on_the_simplex():
    """Learned π (reading P1): m_step_pi must maximise Σ_t Σ_c q_tc log π_c over the
    probability simplex — checked against scipy's constrained optimiser and 2000 Dirichlet points."""
    import scipy.optimize
    rng = np.random.default_rng(11)
    q = rng.dirichlet(np.ones(4) * 0.7, size=9)          # 9 tasks × 4 clusters, rows sum to 1
    f = lambda p: float(np.sum(q * np.log(p)))
    pi = O.m_step_pi(q)
    assert pi.shape == (4,) and abs(pi.sum() - 1.0) < 1e-15 and np.all(pi > 0)
    res = scipy.optimize.minimize(lambda p: -f(p), np.full(4, 0.25), method="SLSQP",
                                  bounds=[(1e-9, 1.0)] * 4, tol=1e-14,
                                  constraints=[{"type": "eq", "fun": lambda p: p.sum() - 1.0}])
    np.testing.assert_allclose(pi, res.x, atol=1e-6)
    others = rng.dirichlet(np.ones(4), size=2000)
    assert f(pi) >= max(f(p) for p in others)
    # one-hot responsibilities: the weights are the cluster fractions (brute count)
    onehot = np.eye(3)[[0, 0, 2, 0, 2, 1, 0, 0]]
    np.testing.assert_array_equal(O.m_step_pi(onehot) * 8, [5, 1, 2])


def test_exact_em_with_learned_pi_likelihood_monotone():
    """EM theory with π learned as well: L(θ) does not decrease, and π
    moves from a lopsided start towards the data's cluster sizes (2 tasks of each cluster)."""
    data = synthetic.small_problem(T=4, C=2, N=12, D=24, sigma=0.1, seed=3, support=3)
    data = dict(data)
    data["pi"] = np.array([0.9, 0.1])
    rng = np.random.default_rng(0)
    alpha0 = rng.uniform(0.0, 1.0, (2, 24)) + 1e-3
    r = O.run(data, 25, mode="exact", alpha0=alpha0, learn_pi=True)
    L = [h["L"] for h in r["history"]]
    assert all(L[i + 1] >= L[i] - 1e-9 * abs(L[i]) for i in range(len(L) - 1))
    assert abs(r["pi"].sum() - 1.0) < 1e-12
    fixed = O.run(data, 25, mode="exact", alpha0=alpha0)
    assert L[-1] >= fixed["history"][-1]["L"] - 1e-9 * abs(L[-1])   # an extra free parameter
    assert abs(r["pi"][0] - 0.5) < abs(0.9 - 0.5)


def test_single_cluster_q_is_one():
    data = synthetic.small_problem(T=3, C=1, N=10, D=20, seed=4)
    e = O.e_step(data, np.ones((1, 20)), 0, mode="cofem", K=4, tol=1e-10, cap=80)
    np.testing.assert_array_equal(e["q"], 1.0)


def test_cofem_converges_to_probe_exact():
    """Tight CG (tol 1e-13, cap 4D): μ and s equal their exact-solve values for the same probes."""
    data = synthetic.small_problem(T=2, C=2, N=10, D=20, seed=5)
    alpha = np.random.default_rng(1).uniform(0.3, 3.0, (2, 20))
    a = O.e_step(data, alpha, 1, mode="cofem", K=5, tol=1e-13, cap=80)
    b = O.e_step(data, alpha, 1, mode="probe_exact", K=5)
    np.testing.assert_allclose(a["mu"], b["mu"], rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(a["s"], b["s"], rtol=1e-8, atol=1e-10)


def test_logdet_estimator_within_ubaru_saad_band():
    """K large, U ≥ bound: |ν̄ − log det Σ| ≤ ε|log det Σ| (ε≈0.21 at K=2000)."""
    data = synthetic.small_problem(T=1, C=1, N=10, D=20, seed=6)
    alpha = np.full((1, 20), 0.7)
    ex = O.e_step(data, alpha, 0, mode="exact")
    co = O.e_step(data, alpha, 0, mode="cofem", K=2000, tol=1e-12, cap=80)
    pe = O.e_step(data, alpha, 0, mode="probe_exact", K=2000)
    assert abs(co["nu"][0, 0] - ex["nu"][0, 0]) <= 0.21 * abs(ex["nu"][0, 0])
    assert co["nu"][0, 0] == pytest.approx(pe["nu"][0, 0], rel=1e-6)
    np.testing.assert_allclose(co["s"][0, 0], ex["s"][0, 0], rtol=0.25)


def test_readout_ties_lowest_and_nmse():
    q = np.array([[0.5, 0.5], [0.2, 0.8]])
    mu = np.arange(2 * 2 * 3, dtype=float).reshape(2, 2, 3)
    a, z = O.readout(q, mu)
    assert list(a) == [0, 1]
    np.testing.assert_array_equal(z, [mu[0, 0], mu[1, 1]])
    assert O.nmse(np.ones(4), 2 * np.ones(4)) == pytest.approx(0.25)


def test_cluster_subset_equals_full_computation():
    """Every (t, c) block of Alg. 2 lines 6-9 is an independent computation: evaluating a subset of
    clusters (used for the full-size sampled parity tests) reproduces the full call's μ, s, ν̄."""
    data = synthetic.small_problem(T=1, C=3, N=10, D=20, K=5, seed=11)
    alpha = np.random.default_rng(3).uniform(0.5, 3.0, (3, 20))
    P = O.probe_signs(9, 0, 1, 0, 3, 5, 20)
    full = O.cofem_task(data["phi"][0], data["y"][0], data["beta"], alpha, data["pi"], P, 1e-8, 80)
    sub = O.cofem_task(data["phi"][0], data["y"][0], data["beta"], alpha, data["pi"], P, 1e-8, 80, clusters=[2, 0])
    for k in ("mu", "s", "nu"):
        np.testing.assert_array_equal(sub[k], full[k][[2, 0]])


# ---------------------------------------------------- partial-Fourier Φ = Ω F ----
def test_partial_fourier_equals_library_fft():
    """Φv = [Re(F v)[rows]; Im(F v)[rows]] with F the unitary DFT: numpy's FFT (pocketfft) of v
    divided by √D, restricted to the sampled rows (the paper's Ω), real-embedded."""
    rng = np.random.default_rng(31)
    for D in (8, 64, 100, 256):
        rows = np.sort(rng.choice(D, size=D // 4, replace=False))
        v = rng.standard_normal(D)
        f = np.fft.fft(v) / math.sqrt(D)
        want = np.concatenate([f.real[rows], f.imag[rows]])
        np.testing.assert_allclose(O.partial_fourier_matrix(D, rows) @ v, want, rtol=0, atol=1e-12)


def test_partial_fourier_dc_row_and_full_mask_unitary():
    """D = 4, Ω = the DC row, v = 1 → Φv = [4/√4, 0] = [2, 0].  Ω = I → ΦᵀΦ = I
    (F unitary: Parseval), the real embedding preserving it."""
    np.testing.assert_allclose(O.partial_fourier_matrix(4, [0]) @ np.ones(4), [2.0, 0.0], atol=1e-15)
    for D in (4, 16, 30):
        P = O.partial_fourier_matrix(D, np.arange(D))
        np.testing.assert_allclose(P.T @ P, np.eye(D), atol=1e-12)


def test_partial_fourier_normal_operator_spectrum():
    """ΦᵀΦ = Re(Fᴴ ΩᵀΩ F) is the circulant whose symbol is m_sym(k) = (m(k) + m(−k mod D))/2 for the
    0/1 mask m of the sampled rows (convolution theorem), so its eigenvalues are exactly the D values
    m_sym(k) ∈ {0, ½, 1} — e.g. frequency k alone (k ≠ 0, D/2) contributes ½ twice."""
    rng = np.random.default_rng(32)
    for D in (16, 64, 90):
        rows = np.sort(rng.choice(D, size=D // 4, replace=False))
        m = np.zeros(D)
        m[rows] = 1.0
        msym = 0.5 * (m + m[(-np.arange(D)) % D])
        P = O.partial_fourier_matrix(D, rows)
        lam = np.linalg.eigvalsh(P.T @ P)
        np.testing.assert_allclose(np.sort(lam), np.sort(msym), atol=1e-12)


def test_partial_fourier_task_data_follow_the_model():
    """Config 6 data (synthetic): y_t − Φ_t z_t is the N(0, σ²) noise of Eq. 1, with
    Φ_t = Ω_t F the oracle's dense real-embedded partial DFT, and the oracle E-step at a tiny D runs
    on it (Φ built from the task's rows)."""
    cfg = synthetic.CONFIGS[6]
    d = synthetic.generate(cfg, [3])
    P = O.partial_fourier_matrix(cfg.D, d["rows"][0])
    res = d["y"][0].astype(np.float64) - P @ d["z"][0]
    assert abs(np.std(res) / cfg.sigma - 1.0) < 0.05 and abs(np.mean(res)) < 5 * cfg.sigma / np.sqrt(res.size)
    small = cfg.replace(D=64, N=16, T=2, support=4, cluster_sizes=(1, 1), C=2)
    ds = synthetic.generate(small)
    e = O.e_step(ds, np.ones((2, 64)), 0, cap=200)
    ex = O.e_step(ds, np.ones((2, 64)), 0, mode="exact")
    np.testing.assert_allclose(e["mu"], ex["mu"], rtol=1e-5, atol=1e-8)
