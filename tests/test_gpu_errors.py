"""Error paths of the C ABI (include/cmtcs.h; SURVEY.md §8(b) error conventions, SPEC.md:123, 141,
289), driven through real inputs rather than debug hooks:

  EBREAKDOWN  dᵀAd ≤ 0 or NaN at Alg. 1 line 3: a NaN in Φ_t makes Ad NaN at the
              first step; the message carries (task, column, step).
  ENUMERIC    ℓ_tc non-finite (Eq. 3): a NaN in y_t reaches ‖y − Φμ‖².
  EEIG        the Lanczos quadrature (Eq. 7-9) on a transcript with γ ≤ 0 (Γ̄ not SPD) or an
              out-of-range step count.
  ESTATE      every call on a context after such a failure.
"""
import re

import numpy as np
import pytest

import synthetic
from gpu_common import make_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_breakdown_reports_task_column_step(torch_cuda):
    from paper_2310_00420_b200 import CmtcsError
    data = synthetic.small_problem(T=3, C=2, N=16, D=32, K=3, seed=21)
    data["phi"][1, 5, 7] = np.nan                # task 1 only
    g = make_gpu(data, cap=50)
    with pytest.raises(CmtcsError, match="EBREAKDOWN") as ei:
        g.em_step(1)
    m = re.search(r"task (\d+), column (-?\d+), step (\d+)", str(ei.value))
    assert m, str(ei.value)
    assert int(m.group(1)) == 1 and int(m.group(3)) == 1      # global task 1, first CG step
    assert ei.value.status == 5
    # the context is unusable afterwards (ESTATE), without another error message
    with pytest.raises(CmtcsError, match="ESTATE"):
        g.em_step(1)
    with pytest.raises(CmtcsError, match="ESTATE"):
        g.posterior()
    g.close()


@pytest.mark.parametrize("engine", ["tensor", "fp32"])
def test_nonfinite_measurements_give_enumeric(torch_cuda, engine):
    from paper_2310_00420_b200 import CmtcsError
    data = synthetic.small_problem(T=2, C=2, N=16, D=32, K=3, seed=22)
    data["y"][0, 3] = np.nan
    g = make_gpu(data, cap=50, engine=engine)
    with pytest.raises(CmtcsError, match="ENUMERIC") as ei:
        g.em_step(1)
    assert ei.value.status == 7 and "task 0" in str(ei.value)
    with pytest.raises(CmtcsError, match="ESTATE"):
        g.em_step(1)
    g.close()


@pytest.mark.parametrize("case", ["negative_gamma", "zero_steps", "steps_past_ld"])
def test_quadrature_failure_gives_eeig(torch_cuda, case):
    import torch
    from paper_2310_00420_b200 import CmtcsError, lanczos_quadrature
    ld = 8
    gam = np.full((2, ld), 0.5)
    xi = np.full((2, ld), 0.3)
    steps = np.array([ld, ld], np.int32)
    if case == "negative_gamma":
        gam[1, 3] = -0.1
    elif case == "zero_steps":
        steps[1] = 0
    else:
        steps[1] = ld + 1
    with pytest.raises(CmtcsError, match="EEIG"):
        lanczos_quadrature(torch.tensor(gam).cuda(), torch.tensor(xi).cuda(),
                           torch.tensor(steps).cuda(), 16)
        torch.cuda.synchronize()


def test_invalid_arguments_leave_context_usable(torch_cuda):
    """EINVAL from argument checking does not break the context (cmtcs.h conventions)."""
    from paper_2310_00420_b200 import CmtcsError
    data = synthetic.small_problem(T=2, C=2, N=16, D=32, K=3, seed=23)
    g = make_gpu(data, cap=50)
    with pytest.raises(CmtcsError, match="EINVAL"):
        g.em_step(0)
    with pytest.raises(CmtcsError, match="EINVAL"):
        g.set_state(np.full((2, 32), -1.0), 0)
    info = g.em_step(1)
    assert np.isfinite(info["loglik"])
    g.close()
