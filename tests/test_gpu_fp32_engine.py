"""Parity of the FP32-CUDA-core operator engine (op_kind = CMTCS_OP_DENSE_FP32, k_simt.cu) with the
fp64 CPU oracle, through the C ABI.

This is the engine the north_star's rule selects where the tensor-core operator's truncating
accumulation breaks a tolerance: every bar here is the north_star's own, L
included (|ΔL| ≤ 1e-3) — the mid-run C3-C5 states are in tests/test_gpu_midrun.py.  Same protocol
as tests/test_gpu_parity.py (cap ×4, mean systems to 1e-10, converged blocks for s).
"""
import re

import numpy as np
import pytest

import synthetic
from oracle import cofem as O
from gpu_common import compare_step, make_gpu, oracle_state, rel_inf, to_np

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


def _single_step(data, alpha, it, cap, tol=None, K=None):
    cfg = data["cfg"]
    K = cfg.K if K is None else K
    tol = cfg.cg_tol if tol is None else tol
    g = make_gpu(data, K=K, tol=tol, cap=cap, alpha=alpha, em_iter0=it, mean_tol=MEAN_TOL, engine="fp32")
    info = g.em_step(1)
    post = to_np(g.posterior())
    steps = g.transcript()["steps"].cpu().numpy().reshape(len(data["tasks"]), -1, K)
    g.close()
    orc = O.e_step(data, alpha, it, mode="cofem", K=K, tol=tol, cap=cap, mu_tol=MEAN_TOL, mu_cap=cap)
    a_next = O.m_step(orc["q"], orc["mu"], orc["s"], alpha)
    conv = np.all(steps < cap, axis=-1) & np.all(orc["probe_steps"].reshape(steps.shape) < cap, axis=-1)
    return post, info, orc, a_next, conv


def _assert_bars(post, info, orc, a_next, conv, label):
    e = compare_step(post, info, orc, a_next, conv)
    print(label, e, "converged", conv.sum(), "/", conv.size)
    assert e["mu"] <= MU_TOL
    assert conv.any() and e["s_conv"] <= S_TOL
    assert np.all(np.abs(post["logdet"] - orc["nu"]) <= nu_tol(orc["nu"]))
    assert e["q_abs"] <= Q_TOL
    assert e["L_abs"] <= L_TOL
    # end-to-end α when q is one-hot to 1e-5 (P-α: every oracle q_tc within 1e-5 of 0 or 1 and the
    # two q's within 1e-5 — with soft q, α_c of a cluster holding a sliver of a task's weight is
    # as sensitive to Δq/q as the M-step's ratio makes it)
    onehot = np.all(np.minimum(orc["q"], 1.0 - orc["q"]) <= 1e-5)
    if onehot and np.max(np.abs(post["q"] - orc["q"])) <= 1e-5:
        assert e["alpha"] <= A_TOL
    return e


@pytest.mark.parametrize("it", [0, 6, 15])
def test_single_step_config1(torch_cuda, it):
    cfg = synthetic.CONFIGS[1]
    data = synthetic.generate(cfg)
    alpha = oracle_state(data, it, mode="cofem")
    post, info, orc, a_next, conv = _single_step(data, alpha, it, cap=4 * cfg.cg_cap)
    assert conv.all()
    _assert_bars(post, info, orc, a_next, conv, f"fp32 engine C1 it {it}")


def test_ragged_shapes(torch_cuda):
    """N, D not multiples of the 128-row tiles or the 8-wide K slabs; P = C·K = 15 columns."""
    data = synthetic.small_problem(T=3, C=3, N=36, D=100, K=5, sigma=0.05, seed=11, support=4)
    alpha = np.random.default_rng(2).uniform(0.2, 5.0, (3, 100))
    post, info, orc, a_next, conv = _single_step(data, alpha, 3, cap=400, tol=1e-7)
    _assert_bars(post, info, orc, a_next, conv, "fp32 engine ragged")


def test_two_column_tiles_and_row_tiles(torch_cuda):
    """P = 16·9 = 144 > one 128-column tile, C = 16 (the maximum), N = 300 and D = 520: several
    ragged row tiles in both stages."""
    data = synthetic.small_problem(T=2, C=16, N=300, D=520, K=9, sigma=0.02, seed=12, support=12)
    alpha = np.random.default_rng(3).uniform(0.3, 3.0, (16, 520))
    post, info, orc, a_next, conv = _single_step(data, alpha, 0, cap=1500, tol=1e-7)
    _assert_bars(post, info, orc, a_next, conv, "fp32 engine C16")


def test_single_step_config2(torch_cuda):
    import torch
    cfg = synthetic.CONFIGS[2]
    data = synthetic.generate(cfg)
    alpha = oracle_state(data, 3, mode="cofem")
    post, info, orc, a_next, conv = _single_step(data, alpha, 3, cap=4 * cfg.cg_cap)
    _assert_bars(post, info, orc, a_next, conv, "fp32 engine C2")
    g = make_gpu(data, cap=4 * cfg.cg_cap, alpha=alpha, em_iter0=3, mean_tol=MEAN_TOL, engine="fp32")
    g.em_step(1, q_override=torch.tensor(orc["q"]).cuda())
    pq = to_np(g.posterior())
    g.close()
    errq = np.max(rel_inf(pq["alpha"], a_next))
    print("fp32 engine C2 q-conditioned alpha", errq)
    assert errq <= A_TOL


@pytest.mark.parametrize("T,C,K", [(3, 2, 4), (3, 3, 3), (4, 4, 33)])
def test_shared_phi_equals_replicated(torch_cuda, T, C, K):
    """One Φ shared by all tasks (the config-5 layout) gives the same result as T copies of it —
    bit for bit: with P = C·K a multiple of 4 the shared-Φ operator runs all tasks' columns as one
    flattened GEMM (column tiles straddle tasks; (4, 33): P = 132, tiles of 128 + ragged), otherwise
    per task (P = 9)."""
    data = synthetic.small_problem(T=T, C=C, N=40, D=96, K=K, seed=18)
    data["phi"][1:] = data["phi"][0]
    a = make_gpu(data, cap=300, engine="fp32")
    a.em_step(2)
    pa = to_np(a.posterior())
    a.close()
    shared = dict(data)
    shared["phi"] = data["phi"][0]
    shared["cfg"] = data["cfg"].replace(shared_phi=True)
    b = make_gpu(shared, cap=300, engine="fp32")
    b.em_step(2)
    pb = to_np(b.posterior())
    b.close()
    for k in ("mu", "s", "logdet", "q", "alpha"):
        np.testing.assert_array_equal(pa[k], pb[k])


def test_full_run_config2(torch_cuda):
    """Config 2's whole run (30 EM iterations from α₀ = 1): identical argmax and |ΔNMSE| ≤ 1e-3
    against the oracle's run (tests/golden/c2_full_run.json, written from oracle/ only)."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "c2_full_run.json")) as f:
        gold = json.load(f)
    cfg = synthetic.CONFIGS[2]
    data = synthetic.generate(cfg)
    g = make_gpu(data, engine="fp32")
    infos = [g.em_step(1) for _ in range(cfg.em_iters)]
    post = to_np(g.posterior())
    g.close()
    nm = O.nmse(post["recon"], data["z"])
    gaps = np.abs(np.array([i["loglik"] for i in infos]) - np.array(gold["L"]))
    print("fp32 engine C2 full run: nmse", nm, gold["nmse"], "|dL|", np.array2string(gaps, precision=2))
    assert list(post["assign"]) == gold["assign"]
    assert abs(nm - gold["nmse"]) <= 1e-3


def test_breakdown_reports_task_column_step(torch_cuda):
    from paper_2310_00420_b200 import CmtcsError
    data = synthetic.small_problem(T=3, C=2, N=16, D=32, K=3, seed=21)
    data["phi"][1, 5, 7] = np.nan                # task 1 only
    g = make_gpu(data, cap=50, engine="fp32")
    with pytest.raises(CmtcsError, match="EBREAKDOWN") as ei:
        g.em_step(1)
    m = re.search(r"task (\d+), column (-?\d+), step (\d+)", str(ei.value))
    assert m and int(m.group(1)) == 1 and int(m.group(3)) == 1, str(ei.value)
    with pytest.raises(CmtcsError, match="ESTATE"):
        g.em_step(1)
    g.close()


def test_engines_agree(torch_cuda):
    """The two dense engines solve the same systems: at C1 their μ agree to the mean tolerance and
    their s, ν̄ to the fp32 probe-CG level."""
    cfg = synthetic.CONFIGS[1]
    data = synthetic.generate(cfg)
    out = {}
    for eng in ("tensor", "fp32"):
        g = make_gpu(data, cap=4 * cfg.cg_cap, mean_tol=MEAN_TOL, engine=eng)
        g.em_step(1)
        out[eng] = to_np(g.posterior())
        g.close()
    assert np.max(rel_inf(out["fp32"]["mu"], out["tensor"]["mu"])) <= 1e-8
    assert np.max(rel_inf(out["fp32"]["s"], out["tensor"]["s"])) <= 1e-4
    assert np.max(np.abs(out["fp32"]["logdet"] - out["tensor"]["logdet"])) <= 5e-3

@pytest.mark.parametrize("T,C,K,N,D", [(5, 2, 16, 96, 160), (6, 4, 20, 132, 300)])
def test_task_halves_bit_identical(torch_cuda, T, C, K, N, D):
    """The two-half CG loops (run_simt_cg) leave every column's arithmetic untouched:
    the posterior of an EM step is bit-identical to the single-loop run (CMTCS_SIMT_SPLIT=0), with
    uneven halves (T = 5: 2 + 3 tasks, P = 32 columns per task; T = 6, P = 80: 2 + 4 — the split must
    land on a 32-column block) and ragged N, D.  The library reads the setting once per process, so
    each mode runs in its own interpreter (tests/split_worker.py)."""
    import json
    import os
    import subprocess
    import sys
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "split_worker.py")
    out = {}
    for mode in ("0", "2"):      # 2: split whatever the size (the default, 1, splits only GPU-filling halves)
        env = dict(os.environ, CMTCS_SIMT_SPLIT=mode)
        r = subprocess.run([sys.executable, worker, *map(str, (T, C, K, N, D))], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[mode] = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["2"]["launches"] > out["0"]["launches"], out       # the split path really ran (12 vs 6 per step)
    assert out["0"]["sha"] == out["2"]["sha"], out
    assert out["0"]["loglik"] == out["2"]["loglik"] and out["0"]["probe_col_iters"] == out["2"]["probe_col_iters"]
