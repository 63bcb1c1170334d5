"""CPU fp64 ORACLE for CoFEM (covariance-free EM, arXiv 2310.00420) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this module.  The product path (paper_2310_00420_b200/) never imports it and shares no code with it.

Plain, slow, obviously-correct NumPy in float64, written from PAPER.md in the paper's order and
notation.  Citations are PAPER.md line numbers (the LaTeX source) with the equation / algorithm:

  Eq. 1   generative model ....................... PAPER.md:24-30
  L(θ)    log-likelihood ......................... PAPER.md:33
  Eq. 3   Σ, μ, q, ℓ (E-step) .................... PAPER.md:45-59
  Eq. 4   α update (M-step) ...................... PAPER.md:61-64
  π update (learned mixture weights) ............. PAPER.md:30 (m_step_pi, reading P1)
  Eq. 5   diagonal estimator s ................... PAPER.md:72-76
  Eq. 6   linear systems A x_k = p_k, A μ = βΦᵀy .. PAPER.md:77-80
  Alg. 1  conjugate gradient ..................... PAPER.md:86-98
  Alg. 2  CoFEM driver ........................... PAPER.md:100-122
  Eq. 7   Lanczos tridiagonal Γ̄ from (γ, ξ) ...... PAPER.md:129-133
  Eq. 8   p'Lp = D Σ_u S²_{u,1} log λ_u ........... PAPER.md:134-138
  Eq. 9   ν̄ = -(1/K) Σ_k Σ_u D S̄²_{u,1} log λ̄_u .... PAPER.md:140-143
  Φ_t = Ω_t F (partial Fourier, §4) ............... PAPER.md:176 (partial_fourier_matrix)

Readings where the paper is silent or ambiguous are DESIGN.md §3 (A-numbers follow SURVEY.md 8(c)):
  A1  ℓ is evaluated in its stationary form ℓ̃ = ℓ - β‖y‖² (identical at the exact μ, see `ell`).
  A2  L(θ̂) is evaluated inside the E-step at the entry state, with the estimated ν̄.
  A5  CG stops after step u when ‖r_{u+1}‖₂ ≤ tol·‖b‖₂, or at the cap.
  A6  Rademacher probes come from the counter hash `probe_signs` (an independent implementation of
      the generator the CUDA side also implements).
  A9/A10 s is clamped at var_floor only inside Eq. 4; α ≤ alpha_max; empty clusters keep α.
  A11 argmax ties go to the lowest cluster index.
Every function below is pinned by tests/test_oracle_pins.py (closed forms, invariants, brute force).
"""
from __future__ import annotations

import math
from typing import Callable, Optional, Sequence

import numpy as np

# --------------------------------------------------------------------------------------------
# Rademacher probes (Alg. 2 line 5; reading A6)
# --------------------------------------------------------------------------------------------
_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def splitmix64_finalize(z: np.ndarray) -> np.ndarray:
    """The splitmix64 output function on uint64 arrays (xorshift 30/27/31, two multiplies)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def probe_word(seed: int, w: np.ndarray) -> np.ndarray:
    """word(w) = mix64(seed + (w+1)·0x9E3779B97F4A7C15 mod 2^64) (reading A6)."""
    w = np.asarray(w, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & _M64) + (w + np.uint64(1)) * np.uint64(_GOLDEN)
    return splitmix64_finalize(z)


def probe_signs(seed: int, it: int, T: int, t: int, C: int, K: int, D: int) -> np.ndarray:
    """p_{it,t,c,k,d} ∈ {+1,-1} as float64 [C, K, D] for global task t at EM iteration `it`.

    Word index w = (((it·T + t)·C + c)·K + k)·⌈D/64⌉ + ⌊d/64⌋; p = +1 iff bit (d mod 64) is 0."""
    nw = (D + 63) // 64
    c = np.arange(C, dtype=np.uint64)[:, None, None]
    k = np.arange(K, dtype=np.uint64)[None, :, None]
    d = np.arange(D, dtype=np.uint64)[None, None, :]
    base = ((np.uint64(it) * np.uint64(T) + np.uint64(t)) * np.uint64(C) + c) * np.uint64(K) + k
    w = base * np.uint64(nw) + d // np.uint64(64)
    bits = (probe_word(seed, w) >> (d % np.uint64(64))) & np.uint64(1)
    return np.where(bits == 0, 1.0, -1.0)


# --------------------------------------------------------------------------------------------
# Operators (A = βΦᵀΦ + diag(α) applied matrix-free)
# --------------------------------------------------------------------------------------------
def normal_apply(phi: np.ndarray, beta: float, alpha_cols: np.ndarray, V: np.ndarray) -> np.ndarray:
    """A V for the columns of V: β Φᵀ(Φ V) + α_col ⊙ V.  alpha_cols is [D, m] (α of each column)."""
    phi = np.asarray(phi, dtype=np.float64)
    return beta * (phi.T @ (phi @ V)) + alpha_cols * V


def partial_fourier_matrix(D: int, rows) -> np.ndarray:
    """Φ = Ω F of the paper's own workload (§4), formed densely (2N × D, real).

    F ∈ ℂ^{D×D} is the unitary DFT, F_{k,d} = exp(−2πi·k·d/D)/√D (reading F1: the unitary
    normalisation); Ω keeps the N rows `rows` of the identity.  z, α and A stay real by
    the real embedding Φ = [Re(ΩF); Im(ΩF)] (reading F1): Φᵀ[u; w] = Re((ΩF)ᴴ(u + iw)),
    so ΦᵀΦ = Re(Fᴴ ΩᵀΩ F).  Written out element by element from the DFT's definition."""
    k = np.asarray(rows, dtype=np.float64)[:, None]
    d = np.arange(D, dtype=np.float64)[None, :]
    ang = -2.0 * np.pi * np.mod(k * d, D) / D
    return np.concatenate([np.cos(ang), np.sin(ang)], axis=0) / math.sqrt(D)


def dense_A(phi: np.ndarray, beta: float, alpha: np.ndarray) -> np.ndarray:
    """A = βΦᵀΦ + diag(α) formed densely (exact modes only)."""
    phi = np.asarray(phi, dtype=np.float64)
    return beta * (phi.T @ phi) + np.diag(alpha)


# --------------------------------------------------------------------------------------------
# Alg. 1 — conjugate gradient, PAPER.md:86-98 (each column of B is its own independent system)
# --------------------------------------------------------------------------------------------
class Breakdown(ArithmeticError):
    """dᵀAd ≤ 0 (non-SPD A or numerical failure); carries the column and step index."""


def conjugate_gradient(apply_A: Callable[[np.ndarray, np.ndarray], np.ndarray], B: np.ndarray,
                       tol: float, cap: int, record: bool = True):
    """Alg. 1 on every column of B (D x m).  apply_A(Dsub, cols) returns A·Dsub for those columns.

    Line 1: x₁ = 0, r₁ = b, d₁ = r₁.   For u = 1, 2, ...:
      line 3 γ_u = r_uᵀr_u / d_uᵀAd_u     line 4 x_{u+1} = x_u + γ_u d_u
      line 5 r_{u+1} = r_u − γ_u A d_u     line 6 ξ_u = r_{u+1}ᵀr_{u+1} / r_uᵀr_u
      line 7 d_{u+1} = r_{u+1} + ξ_u d_u
    A column stops after step u once ‖r_{u+1}‖ ≤ tol·‖b‖ (reading A5) or at u = cap; a zero
    right-hand side takes 0 steps (x = 0).  Returns dict(x, gamma[cap, m], xi[cap, m], steps[m],
    relres[m]) with γ, ξ NaN-padded past each column's steps.
    """
    B = np.asarray(B, dtype=np.float64)
    Dn, m = B.shape
    X = np.zeros_like(B)
    R = B.copy()
    Dv = R.copy()
    rr = np.einsum("ij,ij->j", R, R)
    bnorm = np.sqrt(rr)
    steps = np.zeros(m, dtype=np.int64)
    gam = np.full((cap, m), np.nan) if record else None
    xis = np.full((cap, m), np.nan) if record else None
    active = bnorm > 0
    for u in range(cap):
        idx = np.nonzero(active)[0]
        if idx.size == 0:
            break
        d = Dv[:, idx]
        W = apply_A(d, idx)
        dAd = np.einsum("ij,ij->j", d, W)
        if np.any(~(dAd > 0)):
            j = idx[np.argmax(~(dAd > 0))]
            raise Breakdown(f"CG breakdown: d'Ad <= 0 at column {j}, step {u + 1}")
        g = rr[idx] / dAd
        X[:, idx] += g * d
        R[:, idx] -= g * W
        rr_new = np.einsum("ij,ij->j", R[:, idx], R[:, idx])
        xi = rr_new / rr[idx]
        Dv[:, idx] = R[:, idx] + xi * d
        if record:
            gam[u, idx] = g
            xis[u, idx] = xi
        rr[idx] = rr_new
        steps[idx] = u + 1
        done = np.sqrt(rr_new) <= tol * bnorm[idx]
        active[idx[done]] = False
    relres = np.where(bnorm > 0, np.sqrt(rr) / np.where(bnorm > 0, bnorm, 1.0), 0.0)
    return dict(x=X, gamma=gam, xi=xis, steps=steps, relres=relres)


# --------------------------------------------------------------------------------------------
# Eq. 7-9 — Lanczos quadrature log-det
# --------------------------------------------------------------------------------------------
def assemble_tridiagonal(gamma: np.ndarray, xi: np.ndarray) -> np.ndarray:
    """Γ̄ (U'×U') from γ_1..γ_U' and ξ_1..ξ_{U'-1} (Eq. 7):
    Γ₁₁ = 1/γ₁,  Γ_uu = 1/γ_u + ξ_{u-1}/γ_{u-1},  Γ_{u,u-1} = Γ_{u-1,u} = √ξ_{u-1}/γ_{u-1}."""
    gamma = np.asarray(gamma, dtype=np.float64)
    U = gamma.size
    if U < 1 or np.any(~(gamma > 0)):
        raise ValueError("assemble_tridiagonal needs U' >= 1 and all gamma > 0")
    G = np.zeros((U, U))
    G[0, 0] = 1.0 / gamma[0]
    for u in range(1, U):
        G[u, u] = 1.0 / gamma[u] + xi[u - 1] / gamma[u - 1]
        G[u, u - 1] = G[u - 1, u] = math.sqrt(xi[u - 1]) / gamma[u - 1]
    return G


def quadrature_term(gamma: np.ndarray, xi: np.ndarray, D: int) -> float:
    """τ = D · Σ_u S̄²_{u,1} log λ̄_u (Eq. 8 on the truncated Γ̄) ≈ pᵀ(log A)p.

    Γ̄ = S̄ᵀ diag(λ̄) S̄ with eigenvectors as the ROWS of S̄, so S̄_{u,1} is the first
    component of the u-th eigenvector; numpy's eigh returns eigenvectors as columns, hence V[0, u]."""
    lam, V = np.linalg.eigh(assemble_tridiagonal(gamma, xi))
    if np.any(~(lam > 0)):
        raise ArithmeticError("non-positive Ritz value in Lanczos quadrature")
    return float(D * np.sum(V[0, :] ** 2 * np.log(lam)))


def estimate_logdet(terms: np.ndarray) -> float:
    """ν̄(Σ) = −(1/K) Σ_k τ_k (Eq. 9; Hutchinson)."""
    return -float(np.mean(terms))


def estimate_diagonal(P: np.ndarray, X: np.ndarray) -> np.ndarray:
    """s = (1/K) Σ_k p_k ⊙ x_k (Eq. 5).  P, X are [K, D]."""
    return np.mean(np.asarray(P, dtype=np.float64) * np.asarray(X, dtype=np.float64), axis=0)


# --------------------------------------------------------------------------------------------
# Eq. 3 — ℓ, responsibilities, log-likelihood;  Eq. 4 — M-step
# --------------------------------------------------------------------------------------------
def ell(nu: float, alpha_c: np.ndarray, beta: float, y: np.ndarray, phi_mu: np.ndarray,
        mu: np.ndarray) -> float:
    """ℓ̃_tc = ν̄ + Σ_d log α_cd − β‖y − Φμ‖² − μᵀdiag(α)μ   (reading A1).

    PAPER.md:59 writes ℓ = log det Σ + Σ log α + β yᵀΦμ.  At the exact μ (Aμ = βΦᵀy),
    β yᵀΦμ = β‖y‖² − β‖y − Φμ‖² − μᵀdiag(α)μ, and β‖y‖² does not depend on c, so the softmax
    of Eq. 3 is unchanged; ℓ̃ = ℓ − β‖y‖² is the form whose error is second order in μ's error."""
    y = np.asarray(y, dtype=np.float64)
    res = y - phi_mu
    return float(nu + np.sum(np.log(alpha_c)) - beta * res @ res - mu @ (alpha_c * mu))


def ell_literal(nu: float, alpha_c: np.ndarray, beta: float, y: np.ndarray, phi_mu: np.ndarray) -> float:
    """ℓ exactly as PAPER.md:59 writes it (diagnostic only)."""
    return float(nu + np.sum(np.log(alpha_c)) + beta * np.asarray(y, np.float64) @ phi_mu)


def responsibilities(ell_t: np.ndarray, pi: np.ndarray) -> np.ndarray:
    """q_t = softmax_c(½ℓ_tc + log π_c) (Eq. 3), max-subtracted."""
    a = 0.5 * np.asarray(ell_t, dtype=np.float64) + np.log(pi)
    if not np.any(np.isfinite(a)):
        raise ArithmeticError("softmax of all -inf")
    e = np.exp(a - np.max(a))
    return e / e.sum()


def task_loglik(ell_t: np.ndarray, pi: np.ndarray, beta: float, N: int) -> float:
    """log p(y_t | θ̂) = logsumexp_c(½ℓ̃_tc + log π_c) + (N/2) log(β/2π)   (readings A1, A2).

    From the determinant lemma and Woodbury on y_t ~ N(0, β⁻¹I + Φ diag(α)⁻¹ Φᵀ):
    log p(y_t|c) = ½ℓ_tc − (β/2)‖y‖² + (N/2)log(β/2π) = ½ℓ̃_tc + (N/2)log(β/2π)."""
    a = 0.5 * np.asarray(ell_t, dtype=np.float64) + np.log(pi)
    mx = np.max(a)
    return float(mx + np.log(np.sum(np.exp(a - mx))) + 0.5 * N * math.log(beta / (2.0 * math.pi)))


def m_step(q: np.ndarray, mu: np.ndarray, s: np.ndarray, alpha_old: np.ndarray,
           alpha_max: float = 1e12, var_floor: float = 1e-12, empty_eps: float = 1e-10) -> np.ndarray:
    """Eq. 4: α̃_cd = Σ_t q_tc / Σ_t q_tc [(μ_tcd)² + Σ_tc,dd], Σ_dd ≈ s (Alg. 2 l.115).

    q [T, C], mu/s [T, C, D].  Readings A9/A10: s clamped at var_floor here only; α ≤ alpha_max;
    a cluster with Σ_t q_tc < empty_eps keeps its previous α."""
    num, den = m_step_sums(q, mu, s, var_floor)
    return m_step_finish(num, den, alpha_old, alpha_max, empty_eps)


def m_step_pi(q: np.ndarray) -> np.ndarray:
    """Mixture-weight M-step when π is learned (π "can also be learned by the model",
    citing the mixture-model EM of McLachlan & Basford): the π-dependent part of the EM surrogate,
    Σ_t Σ_c q_tc log π_c, is maximised on the simplex by π_c = (1/T) Σ_t q_tc (reading P1)."""
    q = np.asarray(q, dtype=np.float64)
    return q.sum(axis=0) / q.shape[0]


def m_step_sums(q, mu, s, var_floor=1e-12):
    """The two sums of Eq. 4 over the tasks given (a rank's shard sums to a partial)."""
    q = np.asarray(q, dtype=np.float64)
    num = q.sum(axis=0)
    den = np.einsum("tc,tcd->cd", q, np.asarray(mu, np.float64) ** 2
                    + np.maximum(np.asarray(s, np.float64), var_floor))
    return num, den


def m_step_finish(num, den, alpha_old, alpha_max=1e12, empty_eps=1e-10):
    alpha_old = np.asarray(alpha_old, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        new = np.minimum(num[:, None] / den, alpha_max)
    return np.where((num < empty_eps)[:, None], alpha_old, new)


# --------------------------------------------------------------------------------------------
# E-steps: cofem (Alg. 2 lines 3-12), exact (Eq. 3 literal), probe_exact (K fixed, U → ∞)
# --------------------------------------------------------------------------------------------
def _phi_of(data, i):
    """Φ_t of the i-th task of `data`: the given matrix, or for a partial-Fourier task
    the dense Ω_t F built from its sampled rows."""
    ph = data["phi"]
    if ph is None:
        return partial_fourier_matrix(data["cfg"].D, data["rows"][i])
    return ph if ph.ndim == 2 else ph[i]


def cofem_task(phi: np.ndarray, y: np.ndarray, beta: float, alpha: np.ndarray, pi: np.ndarray,
               P: np.ndarray, tol: float, cap: int, mu_tol: Optional[float] = None,
               mu_cap: Optional[int] = None, clusters: Optional[Sequence[int]] = None) -> dict:
    """Alg. 2 lines 4-12 for one task t and every cluster c.

    P: probes [C, K, D] (line 5).  Line 6: CG on A_tc μ = βΦᵀy and A_tc x_k = p_k.  mu_tol/mu_cap
    optionally solve the mean system to a different tolerance (parity protocol).
    clusters: evaluate lines 6-9 (μ, s, ν̄) for these clusters only — every (t, c) block is an
    independent computation; q and the log-likelihood (line 10) need all clusters and are omitted."""
    if clusters is not None:
        sel = np.asarray(list(clusters), dtype=np.int64)
        full = cofem_task(phi, y, beta, alpha[sel], np.full(sel.size, 1.0 / sel.size), P[sel], tol, cap,
                          mu_tol, mu_cap)
        return {k: full[k] for k in ("mu", "s", "nu", "tau", "mu_steps", "probe_steps", "gamma", "xi")}
    phi64 = np.asarray(phi, dtype=np.float64)
    C, K, Dn = P.shape
    N = phi64.shape[0]
    b = beta * (phi64.T @ np.asarray(y, np.float64))            # Eq. 6 right-hand side βΦᵀy
    # columns: [μ_0 .. μ_{C-1} | probes of c=0 (K) | probes of c=1 | ...]
    col_c = np.concatenate([np.arange(C), np.repeat(np.arange(C), K)])
    alpha_cols = alpha[col_c].T                                   # [D, m]

    def apply_A(Vsub, cols):
        return normal_apply(phi64, beta, alpha_cols[:, cols], Vsub)

    Bp = P.reshape(C * K, Dn).T
    if mu_tol is None and mu_cap is None:
        cg = conjugate_gradient(apply_A, np.concatenate([np.repeat(b[:, None], C, 1), Bp], 1), tol, cap)
        mu = cg["x"][:, :C].T
        Xp = cg["x"][:, C:]
        gam, xis, steps = cg["gamma"][:, C:], cg["xi"][:, C:], cg["steps"]
        mu_steps = steps[:C]
        p_steps = steps[C:]
    else:
        cgm = conjugate_gradient(lambda V, cols: apply_A(V, cols), np.repeat(b[:, None], C, 1),
                                 tol if mu_tol is None else mu_tol, cap if mu_cap is None else mu_cap,
                                 record=False)
        cgp = conjugate_gradient(lambda V, cols: apply_A(V, cols + C), Bp, tol, cap)
        mu = cgm["x"].T
        Xp = cgp["x"]
        gam, xis = cgp["gamma"], cgp["xi"]
        mu_steps, p_steps = cgm["steps"], cgp["steps"]
    Xp = Xp.T.reshape(C, K, Dn)
    s = np.stack([estimate_diagonal(P[c], Xp[c]) for c in range(C)])          # line 7, Eq. 5
    tau = np.zeros((C, K))
    for c in range(C):                                                         # lines 8-9, Eq. 7-9
        for k in range(K):
            j = c * K + k
            U = int(p_steps[j])
            tau[c, k] = quadrature_term(gam[:U, j], xis[:U, j], Dn)
    nu = np.array([estimate_logdet(tau[c]) for c in range(C)])
    phi_mu = (phi64 @ mu.T).T                                                  # Φ μ_tc, [C, N]
    ell_t = np.array([ell(nu[c], alpha[c], beta, y, phi_mu[c], mu[c]) for c in range(C)])
    ell_lit = np.array([ell_literal(nu[c], alpha[c], beta, y, phi_mu[c]) for c in range(C)])
    q = responsibilities(ell_t, pi)                                            # line 10, Eq. 3
    return dict(mu=mu, s=s, nu=nu, tau=tau, ell=ell_t, ell_literal=ell_lit, q=q,
                ll=task_loglik(ell_t, pi, beta, N), mu_steps=mu_steps, probe_steps=p_steps,
                gamma=gam, xi=xis)


def exact_task(phi, y, beta, alpha, pi) -> dict:
    """Eq. 3 literally, with dense factorisations (the O(D³) EM baseline)."""
    phi64 = np.asarray(phi, dtype=np.float64)
    N = phi64.shape[0]
    C = alpha.shape[0]
    b = beta * (phi64.T @ np.asarray(y, np.float64))
    mu, s, nu = [], [], []
    for c in range(C):
        A = dense_A(phi64, beta, alpha[c])
        L = np.linalg.cholesky(A)
        Sigma = np.linalg.inv(A)
        mu.append(Sigma @ b)
        s.append(np.diag(Sigma).copy())
        nu.append(-2.0 * np.sum(np.log(np.diag(L))))                          # log det Σ
    mu, s, nu = np.array(mu), np.array(s), np.array(nu)
    phi_mu = (phi64 @ mu.T).T
    ell_t = np.array([ell(nu[c], alpha[c], beta, y, phi_mu[c], mu[c]) for c in range(C)])
    q = responsibilities(ell_t, pi)
    return dict(mu=mu, s=s, nu=nu, ell=ell_t, q=q, ll=task_loglik(ell_t, pi, beta, N))


def probe_exact_task(phi, y, beta, alpha, pi, P) -> dict:
    """The U → ∞ limit of the covariance-free estimators for the given probes P [C, K, D]:
    x_k = A⁻¹p_k exactly, s by Eq. 5, ν = −(1/K) Σ_k p_kᵀ log(A) p_k via eigh(A)."""
    phi64 = np.asarray(phi, dtype=np.float64)
    N = phi64.shape[0]
    C, K, Dn = P.shape
    b = beta * (phi64.T @ np.asarray(y, np.float64))
    mu, s, nu = [], [], []
    for c in range(C):
        lam, V = np.linalg.eigh(dense_A(phi64, beta, alpha[c]))
        Ainv = (V / lam) @ V.T
        logA = (V * np.log(lam)) @ V.T
        mu.append(Ainv @ b)
        X = (Ainv @ P[c].T).T
        s.append(estimate_diagonal(P[c], X))
        nu.append(-np.mean(np.einsum("kd,de,ke->k", P[c], logA, P[c])))
    mu, s, nu = np.array(mu), np.array(s), np.array(nu)
    phi_mu = (phi64 @ mu.T).T
    ell_t = np.array([ell(nu[c], alpha[c], beta, y, phi_mu[c], mu[c]) for c in range(C)])
    q = responsibilities(ell_t, pi)
    return dict(mu=mu, s=s, nu=nu, ell=ell_t, q=q, ll=task_loglik(ell_t, pi, beta, N))


def e_step(data: dict, alpha: np.ndarray, it: int, mode: str = "cofem", K: Optional[int] = None,
           tol: Optional[float] = None, cap: Optional[int] = None, probe_seed: Optional[int] = None,
           T_global: Optional[int] = None, mu_tol=None, mu_cap=None, probes=None) -> dict:
    """Alg. 2 lines 3-13 over the tasks in `data` at (global) EM iteration `it`."""
    cfg = data["cfg"]
    K = cfg.K if K is None else K
    tol = cfg.cg_tol if tol is None else tol
    cap = cfg.cg_cap if cap is None else cap
    seed = cfg.probe_seed if probe_seed is None else probe_seed
    Tg = cfg.T if T_global is None else T_global
    beta, pi = data["beta"], data["pi"]
    C = alpha.shape[0]
    Dn = alpha.shape[1]
    out = []
    for i, t in enumerate(data["tasks"]):
        phi_t, y_t = _phi_of(data, i), data["y"][i]
        if mode == "exact":
            out.append(exact_task(phi_t, y_t, beta, alpha, pi))
            continue
        P = probes[i] if probes is not None else probe_signs(seed, it, Tg, int(t), C, K, Dn)
        if mode == "probe_exact":
            out.append(probe_exact_task(phi_t, y_t, beta, alpha, pi, P))
        elif mode == "cofem":
            out.append(cofem_task(phi_t, y_t, beta, alpha, pi, P, tol, cap, mu_tol, mu_cap))
        else:
            raise ValueError(mode)
    res = {k: np.array([o[k] for o in out]) for k in ("mu", "s", "nu", "ell", "q", "ll")}
    if mode == "cofem":
        for k in ("mu_steps", "probe_steps", "tau", "ell_literal"):
            res[k] = np.array([o[k] for o in out])
    res["L"] = float(np.mean(res["ll"]))                    # L(θ̂) = (1/T) Σ_t log p(y_t|θ̂)
    res["per_task"] = out
    return res


def readout(q: np.ndarray, mu: np.ndarray):
    """Alg. 2 lines 17-20: a_t = argmax_c q_tc (ties → lowest index, A11); ẑ_t = μ_{t,a_t}."""
    a = np.argmax(q, axis=1)
    return a, mu[np.arange(mu.shape[0]), a]


def nmse(zhat: np.ndarray, z: np.ndarray) -> float:
    """‖ẑ − z̃‖² / ‖z̃‖² over the concatenated tasks (A18; PAPER.md:179 uses the unsquared ratio)."""
    return float(np.sum((zhat - z) ** 2) / np.sum(z ** 2))


def run(data: dict, iters: int, mode: str = "cofem", alpha0: Optional[np.ndarray] = None,
        em_iter0: int = 0, alpha_max=1e12, var_floor=1e-12, empty_eps=1e-10, callback=None,
        learn_pi: bool = False, **kw) -> dict:
    """Alg. 2: `iters` EM iterations from α₀, then the readout.

    The readout uses q and μ of the last E-step (reading A3).  learn_pi: π is updated with α in
    every M-step (m_step_pi, reading P1); the E-step of iteration i uses the π of iteration i − 1."""
    alpha = np.array(data["alpha0"] if alpha0 is None else alpha0, dtype=np.float64)
    data = dict(data)
    data["pi"] = np.array(data["pi"], dtype=np.float64)
    hist = []
    e = None
    for i in range(iters):
        e = e_step(data, alpha, em_iter0 + i, mode, **kw)
        alpha_new = m_step(e["q"], e["mu"], e["s"], alpha, alpha_max, var_floor, empty_eps)
        hist.append(dict(L=e["L"], q=e["q"], alpha_in=alpha, pi_in=data["pi"]))
        if callback is not None:
            callback(i, e, alpha_new)
        alpha = alpha_new
        if learn_pi:
            data["pi"] = m_step_pi(e["q"])
    a, zhat = readout(e["q"], e["mu"])
    return dict(alpha=alpha, pi=data["pi"], assign=a, zhat=zhat, last=e, history=hist,
                nmse=nmse(zhat, data["z"]) if "z" in data else None)
