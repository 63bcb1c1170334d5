"""Helpers for the GPU parity tests: run the CUDA path (through the C ABI) and the oracle on the
same seeded inputs, and compare with the north_star's relative-error measure."""
from __future__ import annotations

import numpy as np

import synthetic
from oracle import cofem as O


def rel_inf(a, b, axis=-1):
    """max_i |a_i − b_i| / max_i |b_i| along `axis` (reading A16)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.max(np.abs(a - b), axis=axis) / np.maximum(np.max(np.abs(b), axis=axis), 1e-300)


def make_gpu(data, *, K=None, tol=None, cap=None, alpha=None, em_iter0=0, task_begin=None, T=None,
             seed=None, mean_tol=-1.0, engine="tensor", learn_pi=False):
    import torch
    from paper_2310_00420_b200 import CoFEM
    cfg = data["cfg"]
    fourier = data.get("phi") is None
    phi = None if fourier else torch.from_numpy(np.ascontiguousarray(data["phi"])).cuda()
    rows = torch.from_numpy(np.ascontiguousarray(data["rows"])).cuda() if fourier else None
    y = torch.from_numpy(np.ascontiguousarray(data["y"])).cuda()
    return CoFEM(phi, y, fourier_rows=rows, D=cfg.D, T=cfg.T if T is None else T, C=data["alpha0"].shape[0],
                 K=cfg.K if K is None else K, beta=data["beta"],
                 cg_max_iters=cfg.cg_cap if cap is None else cap,
                 cg_rel_tol=cfg.cg_tol if tol is None else tol,
                 probe_seed=cfg.probe_seed if seed is None else seed, pi=data["pi"],
                 alpha0=data["alpha0"] if alpha is None else alpha,
                 task_begin=int(data["tasks"][0]) if task_begin is None else task_begin,
                 shared_phi=cfg.shared_phi, em_iter0=em_iter0, mean_rel_tol=mean_tol, engine=engine,
                 learn_pi=learn_pi)


def to_np(post):
    return {k: v.detach().cpu().numpy() for k, v in post.items()}


def oracle_state(data, iters, mode="exact", alpha0=None):
    """An asymmetric EM state reached by the oracle itself (used as the common entry state)."""
    if iters == 0:
        return np.array(data["alpha0"] if alpha0 is None else alpha0, np.float64)
    return O.run(data, iters, mode=mode, alpha0=alpha0)["alpha"]


def compare_step(gpu_post, gpu_info, orc, alpha_next_oracle, converged_mask=None):
    """Returns the error summary of one EM step (GPU vs oracle) as a dict of floats."""
    out = {}
    out["mu"] = float(np.max(rel_inf(gpu_post["mu"], orc["mu"])))
    sm = rel_inf(gpu_post["s"], orc["s"])
    out["s_all"] = float(np.max(sm))
    if converged_mask is not None and converged_mask.any():
        out["s_conv"] = float(np.max(sm[converged_mask]))
    out["nu_abs"] = float(np.max(np.abs(gpu_post["logdet"] - orc["nu"])))
    out["q_abs"] = float(np.max(np.abs(gpu_post["q"] - orc["q"])))
    out["alpha"] = float(np.max(rel_inf(gpu_post["alpha"], alpha_next_oracle)))
    out["inv_alpha"] = float(np.max(rel_inf(1.0 / gpu_post["alpha"], 1.0 / alpha_next_oracle)))
    out["L_abs"] = abs(gpu_info["loglik"] - orc["L"])
    return out
