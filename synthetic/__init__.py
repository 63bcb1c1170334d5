"""Seeded synthetic inputs shaped like the paper's workloads (shared by oracle, tests and bench).

This module holds NO arithmetic of the method (no CG, no estimators, no EM). It only draws the
data of the generative model, PAPER.md:24-30 (Sec. 2, Eq. 1):

    a_t ~ Categorical(pi),   z_t | a_t=c ~ sparse signal on cluster c's support,
    y_t = Phi_t z_t + eps_t, eps_t ~ N(0, sigma^2 I),  beta = 1/sigma^2.

The five configurations are the ones BASELINE.json lists (configs[0..4]); the paper's own
Sec. 4 workload (partial DFT Phi) is replaced there by i.i.d. Gaussian Phi with the
same N = D/4 ratio on C2-C5.  Every array is a deterministic function of
(root seed, config id, stream, task index), so any task subset (a rank's shard) can be generated
on its own and is bit-identical to the same tasks of the full set.

Streams of numpy.random.SeedSequence([ROOT, cfg_id, stream, t]):
    0 supports (per config, t = 0)      1 Phi_t (t = task; shared Phi uses t = 0)
    2 nonzero values of z_t             3 noise eps_t            4 task labels (t = 0)
    5 sampled Fourier rows of task t (partial-Fourier configs)

Config 6 is the paper's own §4 workload: Phi_t = Omega_t F, the unitary DFT F
undersampled by a random row mask Omega_t per task (N = D/4 rows), real-embedded as
[Re(Omega_t F); Im(Omega_t F)] (reading F1), 5 % sparse N(0,1) signals, sigma = 0.05.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, Optional, Sequence

import numpy as np

ROOT_SEED = 231000420


@dataclasses.dataclass(frozen=True)
class Config:
    cfg_id: int
    name: str
    T: int
    C: int
    N: int
    D: int
    K: int
    sigma: float
    em_iters: int
    cg_cap: int
    cg_tol: float
    cluster_sizes: tuple          # true cluster sizes (sum = T)
    support: int                  # support size per true cluster
    overlap_core: int = 0         # indices shared by every cluster's support (C2: 20 % overlap)
    values: str = "normal"        # "normal": N(0,1) nonzeros; "sign": +-1 with random sign
    shared_phi: bool = False      # C5: one Phi for all tasks
    operator: str = "dense"       # "dense": Phi_t given as a matrix; "fourier": Phi_t = Omega_t F (C6)

    @property
    def beta(self) -> float:
        return 1.0 / (self.sigma * self.sigma)

    @property
    def M(self) -> int:
        """Right-hand sides per task: C*(K+1) (1 mean column + K probes per cluster)."""
        return self.C * (self.K + 1)

    @property
    def probe_seed(self) -> int:
        return ROOT_SEED * 16 + self.cfg_id

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs[0..4]; cfg_id = index + 1.
CONFIGS: Dict[int, Config] = {
    1: Config(1, "C1-tiny", T=4, C=2, N=32, D=64, K=8, sigma=0.01, em_iters=20, cg_cap=64,
              cg_tol=1e-6, cluster_sizes=(2, 2), support=4),
    2: Config(2, "C2", T=16, C=4, N=256, D=1024, K=20, sigma=0.01, em_iters=30, cg_cap=200,
              cg_tol=1e-6, cluster_sizes=(4, 4, 4, 4), support=30, overlap_core=6),
    3: Config(3, "C3", T=64, C=4, N=1024, D=4096, K=20, sigma=0.005, em_iters=30, cg_cap=300,
              cg_tol=1e-6, cluster_sizes=(32, 16, 8, 8), support=100),
    4: Config(4, "C4", T=256, C=8, N=2048, D=8192, K=32, sigma=0.01, em_iters=20, cg_cap=400,
              cg_tol=1e-6, cluster_sizes=(32,) * 8, support=200, values="sign"),
    5: Config(5, "C5-sharedPhi", T=512, C=16, N=4096, D=16384, K=20, sigma=0.01, em_iters=10,
              cg_cap=300, cg_tol=1e-6, cluster_sizes=(32,) * 16, support=400, shared_phi=True),
    # the paper's §4 workload: partial DFT, N = D/4 sampled rows, 5 % support,
    # sigma = 0.05, K = 15 probes, U = 50 CG steps; T/C in the range of Fig. 1(e, f)
    6: Config(6, "C6-partialFourier", T=64, C=4, N=2048, D=8192, K=15, sigma=0.05, em_iters=30,
              cg_cap=50, cg_tol=1e-6, cluster_sizes=(16,) * 4, support=410, operator="fourier"),
}


def _rng(cfg: Config, stream: int, t: int = 0) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([ROOT_SEED, cfg.cfg_id, stream, t]))


def supports(cfg: Config) -> list:
    """Support index sets of the true clusters (SURVEY.md A19 reading of PAPER.md:178-179)."""
    rng = _rng(cfg, 0)
    nclu = len(cfg.cluster_sizes)
    if cfg.overlap_core > 0:
        # a core shared by all clusters plus disjoint private parts (C2: "20 % overlap")
        n_priv = cfg.support - cfg.overlap_core
        perm = rng.permutation(cfg.D)
        core = perm[: cfg.overlap_core]
        out = []
        for j in range(nclu):
            priv = perm[cfg.overlap_core + j * n_priv: cfg.overlap_core + (j + 1) * n_priv]
            out.append(np.sort(np.concatenate([core, priv])))
        return out
    return [np.sort(rng.choice(cfg.D, size=cfg.support, replace=False)) for _ in range(nclu)]


def labels(cfg: Config) -> np.ndarray:
    """True cluster label of every task: a seeded permutation of the cluster blocks (A20)."""
    lab = np.concatenate([np.full(s, j, dtype=np.int32) for j, s in enumerate(cfg.cluster_sizes)])
    assert lab.size == cfg.T
    return lab[_rng(cfg, 4).permutation(cfg.T)]


def phi(cfg: Config, t: int) -> np.ndarray:
    """Phi_t: N x D, i.i.d. N(0, 1/N) drawn as fp32(standard normal) * fp32(1/sqrt(N)) (A21)."""
    g = _rng(cfg, 1, 0 if cfg.shared_phi else t)
    a = g.standard_normal(size=(cfg.N, cfg.D), dtype=np.float32)
    a *= np.float32(1.0 / math.sqrt(cfg.N))
    return a


def fourier_rows(cfg: Config, t: int) -> np.ndarray:
    """Omega_t: N distinct DFT rows of [0, D), drawn uniformly per task, sorted."""
    return np.sort(_rng(cfg, 5, t).choice(cfg.D, size=cfg.N, replace=False)).astype(np.int32)


def fourier_measure(cfg: Config, rows: np.ndarray, z: np.ndarray) -> np.ndarray:
    """The forward model Phi_t z for Phi_t = [Re(Omega F); Im(Omega F)], F the unitary DFT (the
    data model of Eq. 1 evaluated with numpy's FFT; fp64)."""
    f = np.fft.fft(z) / math.sqrt(cfg.D)
    return np.concatenate([f.real[rows], f.imag[rows]])


def z_true(cfg: Config, t: int, sup=None, lab=None) -> np.ndarray:
    sup = supports(cfg) if sup is None else sup
    lab = labels(cfg) if lab is None else lab
    s = sup[int(lab[t])]
    g = _rng(cfg, 2, t)
    z = np.zeros(cfg.D, dtype=np.float64)
    if cfg.values == "sign":
        z[s] = np.where(g.random(s.size) < 0.5, -1.0, 1.0)
    else:
        z[s] = g.standard_normal(s.size)
    return z


def measurements(cfg: Config, t: int, phi_t: np.ndarray, z: np.ndarray) -> np.ndarray:
    """y_t = fp32(Phi_t z_t + eps_t), computed in fp64 then rounded once (A21).  phi_t may be given
    already widened to fp64 (the shared-Phi config widens it once for all tasks)."""
    eps = _rng(cfg, 3, t).standard_normal(cfg.N) * cfg.sigma
    p64 = phi_t if phi_t.dtype == np.float64 else phi_t.astype(np.float64)
    return (p64 @ z + eps).astype(np.float32)


def generate(cfg: Config, tasks: Optional[Sequence[int]] = None) -> dict:
    """Data of the tasks in `tasks` (default: all).  Returns a dict:

    phi   float32 [T_sel, N, D]   (shared_phi: [N, D]; None for the partial-Fourier config, whose
                                   Phi_t is given by `rows` int32 [T_sel, N] and y has 2N entries)
    y     float32 [T_sel, N]
    z     float64 [T_sel, D]      true signals
    labels int32  [T_sel]         true clusters
    tasks int64   [T_sel]         global task indices
    beta, pi (float64 [C]), alpha0 (float64 [C, D], all ones: A4), cfg
    """
    tasks = np.arange(cfg.T) if tasks is None else np.asarray(list(tasks), dtype=np.int64)
    sup = supports(cfg)
    lab = labels(cfg)
    if cfg.operator == "fourier":
        rows = np.stack([fourier_rows(cfg, int(t)) for t in tasks])
        zs = np.stack([z_true(cfg, int(t), sup, lab) for t in tasks])
        ys = np.stack([(fourier_measure(cfg, rows[i], zs[i])
                        + _rng(cfg, 3, int(t)).standard_normal(2 * cfg.N) * cfg.sigma).astype(np.float32)
                       for i, t in enumerate(tasks)])
        return dict(phi=None, rows=rows, y=ys, z=zs, labels=lab[tasks], tasks=tasks, beta=cfg.beta,
                    pi=np.full(cfg.C, 1.0 / cfg.C), alpha0=np.ones((cfg.C, cfg.D)), cfg=cfg)
    if cfg.shared_phi:
        ph = phi(cfg, 0)
        ph64 = ph.astype(np.float64)
        phis = None
    else:
        phis = np.empty((len(tasks), cfg.N, cfg.D), dtype=np.float32)
    ys = np.empty((len(tasks), cfg.N), dtype=np.float32)
    zs = np.empty((len(tasks), cfg.D), dtype=np.float64)
    for i, t in enumerate(tasks):
        p = ph64 if cfg.shared_phi else phi(cfg, int(t))
        if not cfg.shared_phi:
            phis[i] = p
        zs[i] = z_true(cfg, int(t), sup, lab)
        ys[i] = measurements(cfg, int(t), p, zs[i])
    return dict(
        phi=ph if cfg.shared_phi else phis,
        y=ys,
        z=zs,
        labels=lab[tasks],
        tasks=tasks,
        beta=cfg.beta,
        pi=np.full(cfg.C, 1.0 / cfg.C),
        alpha0=np.ones((cfg.C, cfg.D)),
        cfg=cfg,
    )


def shard(T: int, rank: int, world: int) -> tuple:
    """Contiguous task block [begin, end) of `rank` among `world` ranks.

    The first T % world ranks get one extra task, so block sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(T, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def small_problem(T=3, C=2, N=12, D=24, K=6, sigma=0.05, seed=7, support=3, cap=None, tol=1e-6,
                  em_iters=3) -> dict:
    """A tiny ad-hoc problem for unit tests (not one of the five configs)."""
    cfg = Config(100 + seed, "adhoc", T=T, C=C, N=N, D=D, K=K, sigma=sigma, em_iters=em_iters,
                 cg_cap=cap if cap is not None else 4 * D, cg_tol=tol,
                 cluster_sizes=tuple([T // C + (1 if j < T % C else 0) for j in range(C)]),
                 support=support)
    return generate(cfg)
