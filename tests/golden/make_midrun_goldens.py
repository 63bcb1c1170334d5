"""Oracle-only goldens for the mid-run parity tests (tests/test_gpu_midrun.py).

Calls only synthetic/ and oracle/ (never the CUDA path).  Every E-step block (t, c) of Alg. 2
lines 6-9 is an independent computation, so this script farms the oracle's
per-task / per-(task, cluster) calls out to worker processes (one BLAS thread each) and assembles
the results exactly as oracle.cofem.e_step / run would (L = mean_t log p(y_t), Eq. 4 via
oracle.cofem.m_step, readout via oracle.cofem.readout).  The arithmetic is the oracle's.

  python tests/golden/make_midrun_goldens.py c3run     C3: the full 30-iteration run (c3_full_run.json,
                                                       c3_states.npz: α at every iteration)
  python tests/golden/make_midrun_goldens.py c3step    C3: one E-step + M-step from the run's α at
                                                       EM iteration 8, all 64 tasks, cap 4×300
  python tests/golden/make_midrun_goldens.py c4state   C4: 5 EM iterations on 8 tasks (one per true
                                                       cluster) from α₀ = 1 → a mid-run α
  python tests/golden/make_midrun_goldens.py c4step    C4: one E-step from that α on tasks [0, 2), cap 4×400
  python tests/golden/make_midrun_goldens.py c5state   C5: 2 EM iterations on 8 tasks (one per even true cluster)
  python tests/golden/make_midrun_goldens.py c5step    C5: one E-step from that α on task 0, cap 4×300
"""
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import multiprocessing as mp  # noqa: E402

import numpy as np  # noqa: E402

import synthetic  # noqa: E402
from oracle import cofem as O  # noqa: E402

MEAN_TOL = 1e-10          # parity protocol P-μ (DESIGN.md §3 A5, §6): mean systems solved to 1e-10
NPROC = int(os.environ.get("GOLDEN_PROCS", str(os.cpu_count() or 8)))


def _task_estep(args):
    """oracle E-step of one task (all clusters): the per-task part of oracle.cofem.e_step."""
    cid, t, alpha, it, cap, mu_tol = args
    cfg = synthetic.CONFIGS[cid]
    data = synthetic.generate(cfg, [t])
    e = O.e_step(data, alpha, it, mode="cofem", cap=cap, mu_tol=mu_tol,
                 mu_cap=None if mu_tol is None else cap)
    r = {k: e[k][0] for k in ("mu", "s", "nu", "ell", "q", "ll", "mu_steps", "probe_steps")}
    return t, r


_DATA = {}


def _task_data(cid, t):
    """synthetic.generate(cfg, [t]) with a per-worker cache (the shared-Φ config draws its 268 MB Φ
    once per worker; the per-task parts come from synthetic's own per-task functions)."""
    cfg = synthetic.CONFIGS[cid]
    if (cid, t) in _DATA:
        return _DATA[(cid, t)]
    if cfg.shared_phi:
        if ("phi", cid) not in _DATA:
            ph = synthetic.phi(cfg, 0)
            _DATA[("phi", cid)] = (ph, ph.astype(np.float64), synthetic.supports(cfg), synthetic.labels(cfg))
        ph, ph64, sup, lab = _DATA[("phi", cid)]
        z = synthetic.z_true(cfg, t, sup, lab)
        data = dict(phi=ph, y=synthetic.measurements(cfg, t, ph64, z)[None], z=z[None], tasks=np.array([t]),
                    beta=cfg.beta, pi=np.full(cfg.C, 1.0 / cfg.C), cfg=cfg)
    else:
        _DATA.clear()
        data = synthetic.generate(cfg, [t])
    _DATA[(cid, t)] = data
    return data


def _block_estep(args):
    """oracle lines 6-9 of one (task, cluster) block (oracle.cofem.cofem_task(..., clusters=[c]))."""
    cid, t, c, alpha, it, cap, mu_tol = args
    cfg = synthetic.CONFIGS[cid]
    data = _task_data(cid, t)
    phi_t = data["phi"] if cfg.shared_phi else data["phi"][0]
    P = O.probe_signs(cfg.probe_seed, it, cfg.T, t, cfg.C, cfg.K, cfg.D)
    o = O.cofem_task(phi_t, data["y"][0], data["beta"], alpha, data["pi"], P, cfg.cg_tol, cap,
                     mu_tol=mu_tol, mu_cap=cap, clusters=[c])
    phi64 = np.asarray(phi_t, np.float64)
    ell = O.ell(o["nu"][0], alpha[c], data["beta"], data["y"][0], phi64 @ o["mu"][0], o["mu"][0])
    return t, c, dict(mu=o["mu"][0], s=o["s"][0], nu=o["nu"][0], ell=ell, probe_steps=np.asarray(o["probe_steps"]),
                      mu_steps=np.asarray(o["mu_steps"]))


def estep_tasks(pool, cid, tasks, alpha, it, cap, mu_tol=None):
    res = dict(pool.map(_task_estep, [(cid, int(t), alpha, it, cap, mu_tol) for t in tasks]))
    out = {k: np.array([res[int(t)][k] for t in tasks]) for k in res[int(tasks[0])]}
    out["L"] = float(np.mean(out["ll"]))
    return out


def estep_blocks(pool, cid, tasks, alpha, it, cap, mu_tol=None):
    """Blocks of every (t, c), then Eq. 3's q and log p(y_t) from the blocks' ℓ (oracle functions)."""
    cfg = synthetic.CONFIGS[cid]
    jobs = [(cid, int(t), c, alpha, it, cap, mu_tol) for t in tasks for c in range(cfg.C)]
    got = {(t, c): r for t, c, r in pool.map(_block_estep, jobs, chunksize=1)}
    out = {k: np.array([[got[(int(t), c)][k] for c in range(cfg.C)] for t in tasks])
           for k in ("mu", "s", "nu", "ell", "probe_steps", "mu_steps")}
    pi = np.full(cfg.C, 1.0 / cfg.C)
    out["q"] = np.array([O.responsibilities(out["ell"][i], pi) for i in range(len(tasks))])
    out["ll"] = np.array([O.task_loglik(out["ell"][i], pi, cfg.beta, cfg.N) for i in range(len(tasks))])
    out["L"] = float(np.mean(out["ll"]))
    return out


def em_run(pool, cid, tasks, iters, alpha0, estep, log):
    """Alg. 2 over `tasks` (oracle.cofem.run's loop: E-step, Eq. 4, readout of the last E-step)."""
    cfg = synthetic.CONFIGS[cid]
    alpha = np.array(alpha0, np.float64)
    states, Ls, caps = [alpha.copy()], [], []
    e = None
    for i in range(iters):
        t0 = time.time()
        e = estep(pool, cid, tasks, alpha, i, cfg.cg_cap)
        alpha = O.m_step(e["q"], e["mu"], e["s"], alpha)
        Ls.append(e["L"])
        caps.append(int(np.sum(np.asarray(e["probe_steps"]) >= cfg.cg_cap)))
        states.append(alpha.copy())
        log(f"{cfg.name} it {i}: L {e['L']:.6f} probe steps max {np.max(e['probe_steps'])} "
            f"cap hits {caps[-1]} ({time.time() - t0:.0f} s)")
    return alpha, np.array(states), Ls, caps, e


def save_step(name, cid, tasks, alpha_in, it, cap, e, extra=None):
    a_next = O.m_step(e["q"], e["mu"], e["s"], alpha_in)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                        tasks=np.asarray(tasks, np.int64), alpha_in=alpha_in, it=it, cap=cap,
                        mean_tol=MEAN_TOL, mu=e["mu"].astype(np.float32), s=e["s"].astype(np.float32),
                        nu=e["nu"], q=e["q"], ll=e["ll"], L=e["L"], alpha_next=a_next,
                        probe_steps=np.asarray(e["probe_steps"]).astype(np.int32),
                        mu_steps=np.asarray(e["mu_steps"]).astype(np.int32), **(extra or {}))


def main(which):
    log = lambda m: print(m, flush=True)  # noqa: E731
    with mp.get_context("fork").Pool(NPROC) as pool:
        if which == "c3run":
            cfg = synthetic.CONFIGS[3]
            tasks = list(range(cfg.T))
            alpha, states, Ls, caps, e = em_run(pool, 3, tasks, cfg.em_iters, np.ones((cfg.C, cfg.D)),
                                                estep_tasks, log)
            assign, zhat = O.readout(e["q"], e["mu"])
            z = synthetic.generate(cfg)["z"]
            out = {"config": cfg.name, "em_iters": cfg.em_iters, "assign": [int(a) for a in assign],
                   "nmse": O.nmse(zhat, z), "L": Ls, "probe_cap_hits": caps,
                   "source": "oracle.cofem per-task E-steps + m_step + readout over all 64 tasks of "
                             "CONFIGS[3], 30 iterations from alpha0 = 1, fp64 (make_midrun_goldens.py c3run)"}
            with open(os.path.join(HERE, "c3_full_run.json"), "w") as f:
                json.dump(out, f, indent=1)
            np.savez_compressed(os.path.join(HERE, "c3_states.npz"), alpha=states[:11])
        elif which == "c3step":
            cfg = synthetic.CONFIGS[3]
            it = 8
            alpha = np.load(os.path.join(HERE, "c3_states.npz"))["alpha"][it]
            e = estep_tasks(pool, 3, list(range(cfg.T)), alpha, it, 4 * cfg.cg_cap, MEAN_TOL)
            save_step("c3_step8", 3, list(range(cfg.T)), alpha, it, 4 * cfg.cg_cap, e)
            log(f"c3 step: L {e['L']} probe steps max {np.max(e['probe_steps'])}")
        elif which in ("c4state", "c5state"):
            cid = 4 if which == "c4state" else 5
            cfg = synthetic.CONFIGS[cid]
            lab = synthetic.labels(cfg)
            tasks = [int(np.nonzero(lab == j)[0][0]) for j in range(len(cfg.cluster_sizes))]
            if cid == 5:
                tasks = tasks[::2]            # C5: 8 of the 16 true clusters (the oracle's cost)
            iters = 5 if cid == 4 else 2
            alpha, states, Ls, caps, e = em_run(pool, cid, tasks, iters, np.ones((cfg.C, cfg.D)),
                                                estep_blocks, log)
            np.savez_compressed(os.path.join(HERE, f"c{cid}_state.npz"), alpha=alpha, it=iters,
                                tasks=np.asarray(tasks), L=np.asarray(Ls), cap_hits=np.asarray(caps))
        elif which in ("c4step", "c5step"):
            cid = 4 if which == "c4step" else 5
            cfg = synthetic.CONFIGS[cid]
            st = np.load(os.path.join(HERE, f"c{cid}_state.npz"))
            alpha, it = st["alpha"], int(st["it"])
            tasks = [0, 1] if cid == 4 else [0]
            e = estep_blocks(pool, cid, tasks, alpha, it, 4 * cfg.cg_cap, MEAN_TOL)
            save_step(f"c{cid}_step{it}", cid, tasks, alpha, it, 4 * cfg.cg_cap, e)
            log(f"c{cid} step: L {e['L']} probe steps max {np.max(e['probe_steps'])}")
        else:
            raise SystemExit(__doc__)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "")
