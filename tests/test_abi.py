"""The C-ABI library loads and exports every symbol include/cmtcs.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "cmtcs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cmtcs_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    f = header_functions()
    for name in ("cmtcs_init", "cmtcs_em_step", "cmtcs_posterior", "cmtcs_get_unique_id",
                 "cmtcs_last_error", "cmtcs_destroy"):
        assert name in f


def test_library_exports_every_declared_symbol():
    import paper_2310_00420_b200.build as b
    b.build()
    lib = ctypes.CDLL(b.LIB)
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_names_match_header():
    from paper_2310_00420_b200 import cmtcs
    assert sorted(cmtcs.EXPORTED) == header_functions()
    for n in cmtcs.EXPORTED:
        assert callable(getattr(cmtcs, n))


def test_struct_layout_matches_c():
    """Compile a tiny C program that prints sizeof/offsetof of the ABI structs; compare to ctypes."""
    import subprocess
    import tempfile
    from paper_2310_00420_b200 import cmtcs
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "cmtcs.h"
int main(void){
  printf("%zu %zu %zu %zu %zu\n", sizeof(cmtcs_problem), offsetof(cmtcs_problem, beta),
         offsetof(cmtcs_problem, probe_seed), offsetof(cmtcs_problem, em_iter0), sizeof(cmtcs_step_info));
  printf("%zu %zu %zu %zu\n", offsetof(cmtcs_step_info, probe_steps_mean), offsetof(cmtcs_step_info, kernel_launches), offsetof(cmtcs_step_info, tile_col_iters),
         offsetof(cmtcs_problem, mean_rel_tol));
  printf("%zu %zu %d %d %zu\n", offsetof(cmtcs_problem, op_kind), offsetof(cmtcs_problem, fourier_rows), (int)CMTCS_OP_PARTIAL_FOURIER,
         (int)CMTCS_OP_DENSE_FP32, offsetof(cmtcs_problem, learn_pi));
  return 0; }
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        out = subprocess.check_output([exe]).decode().split()
    P, S = cmtcs.cmtcs_problem, cmtcs.cmtcs_step_info
    want = [ctypes.sizeof(P), P.beta.offset, P.probe_seed.offset, P.em_iter0.offset, ctypes.sizeof(S),
            S.probe_steps_mean.offset, S.kernel_launches.offset, S.tile_col_iters.offset, P.mean_rel_tol.offset,
            P.op_kind.offset, P.fourier_rows.offset, cmtcs.CMTCS_OP_PARTIAL_FOURIER, cmtcs.CMTCS_OP_DENSE_FP32,
            P.learn_pi.offset]
    assert [int(x) for x in out] == want


def test_invalid_problem_rejected_without_gpu():
    from paper_2310_00420_b200 import cmtcs
    import numpy as np
    pi = np.array([0.5, 0.5])
    p = cmtcs.cmtcs_problem(T=4, N=30, D=64, C=2, K=3, beta=1.0, pi=pi.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                            cg_max_iters=10, cg_rel_tol=1e-6, alpha_max=1e12, var_floor=1e-12, empty_eps=1e-10,
                            probe_seed=1, task_begin=0, task_end=4)
    with pytest.raises(cmtcs.CmtcsError, match="EINVAL"):
        cmtcs.cmtcs_workspace_size(p)            # N % 4 != 0
    p.N = 32
    assert cmtcs.cmtcs_workspace_size(p) > 0
    p.C = 17
    with pytest.raises(cmtcs.CmtcsError, match="EINVAL"):
        cmtcs.cmtcs_workspace_size(p)
    p.C = 2
    p.op_kind = cmtcs.CMTCS_OP_DENSE_FP32        # the FP32-engine workspace has no Φᵀ / tf32 pairs
    ws_fp32 = cmtcs.cmtcs_workspace_size(p)
    p.op_kind = cmtcs.CMTCS_OP_DENSE
    assert 0 < ws_fp32 < cmtcs.cmtcs_workspace_size(p)
    p.op_kind = 3
    with pytest.raises(cmtcs.CmtcsError, match="EINVAL"):
        cmtcs.cmtcs_workspace_size(p)
    p.op_kind = cmtcs.CMTCS_OP_DENSE
    pi[0] = 0.7
    with pytest.raises(cmtcs.CmtcsError, match="EINVAL"):
        cmtcs.cmtcs_workspace_size(p)
    pi[0] = 0.5
    p.learn_pi = 2                               # learn_pi is a 0/1 switch
    with pytest.raises(cmtcs.CmtcsError, match="EINVAL"):
        cmtcs.cmtcs_workspace_size(p)
    p.learn_pi = 1
    assert cmtcs.cmtcs_workspace_size(p) > 0
