"""User-facing wrapper: a CoFEM run whose device memory is owned by PyTorch tensors.

All arithmetic happens in libcmtcs.so (see cmtcs.py); this class only allocates tensors, passes
their pointers and the current CUDA stream, and converts results back to tensors.
"""
from __future__ import annotations

import numpy as np
import torch

from . import cmtcs as _c


class CoFEM:
    """One rank's share of a clustered multi-task CS problem fit by CoFEM (Alg. 2).

    phi: cuda fp32 [T_loc, N, D] (or [N, D] with shared_phi), y: cuda fp32 [T_loc, N].
    Tasks of this rank are global tasks task_begin .. task_begin + T_loc - 1 of T.
    Partial-Fourier sensing (the paper's §4 workload): phi=None, fourier_rows = cuda
    int32 [T_loc, N] sampled DFT rows, y = cuda fp32 [T_loc, 2N] (real parts, then imaginary), D given.
    engine (dense Φ only): "fp32" (default) — the operator on the FP32 CUDA cores (round-to-nearest
    accumulation, CMTCS_OP_DENSE_FP32), the path that meets every north_star tolerance (DESIGN.md §3
    reading E1, §6); "tensor" — on the tcgen05 tensor cores (3xTF32, one persistent kernel), 2-3x
    faster, |ΔL| above 1e-3 at configs 4-5.
    """

    def __init__(self, phi: torch.Tensor, y: torch.Tensor, *, T: int, C: int, K: int, beta: float,
                 cg_max_iters: int, cg_rel_tol: float, probe_seed: int, pi=None, alpha0=None,
                 task_begin: int = 0, shared_phi: bool = False, em_iter0: int = 0,
                 alpha_max: float = 1e12, var_floor: float = 1e-12, empty_eps: float = 1e-10,
                 mean_rel_tol: float = -1.0,
                 nccl_uid: bytes | None = None, rank: int = 0, world: int = 1, stream=None,
                 fourier_rows: torch.Tensor | None = None, D: int | None = None, engine: str = "fp32",
                 learn_pi: bool = False):
        fourier = fourier_rows is not None
        if engine not in ("tensor", "fp32"):
            raise ValueError(f"engine must be 'tensor' or 'fp32', got {engine!r}")
        if not (y.is_cuda and (fourier_rows.is_cuda if fourier else phi.is_cuda)):
            raise ValueError("phi (or fourier_rows) and y must be CUDA tensors (no CPU path exists)")
        self.y = y.contiguous() if y.dtype == torch.float32 else y.float().contiguous()
        self.device = self.y.device
        T_loc = self.y.shape[0]
        if fourier:
            self.phi = None
            self.rows = fourier_rows.to(torch.int32).contiguous()
            N = self.rows.shape[1]
            if D is None:
                raise ValueError("the partial-Fourier operator needs D")
        else:
            self.phi = phi.contiguous() if phi.dtype == torch.float32 else phi.float().contiguous()
            self.rows = None
            N = self.y.shape[1]
            D = self.phi.shape[-1]
        self.T, self.T_loc, self.N, self.D, self.C, self.K = T, T_loc, N, D, C, K
        self._pi = np.ascontiguousarray(np.full(C, 1.0 / C) if pi is None else np.asarray(pi, np.float64))
        self.problem = _c.cmtcs_problem(
            T=T, N=N, D=D, C=C, K=K, shared_phi=int(bool(shared_phi)), beta=float(beta),
            pi=self._pi.ctypes.data_as(_c.POINTER(_c.c_double)), cg_max_iters=int(cg_max_iters),
            cg_rel_tol=float(cg_rel_tol), alpha_max=float(alpha_max), var_floor=float(var_floor),
            empty_eps=float(empty_eps), probe_seed=int(probe_seed) & ((1 << 64) - 1),
            task_begin=int(task_begin), task_end=int(task_begin) + T_loc, em_iter0=int(em_iter0),
            mean_rel_tol=float(mean_rel_tol),
            op_kind=_c.CMTCS_OP_PARTIAL_FOURIER if fourier else
            (_c.CMTCS_OP_DENSE_FP32 if engine == "fp32" else _c.CMTCS_OP_DENSE),
            fourier_rows=self.rows.data_ptr() if fourier else None, learn_pi=int(bool(learn_pi)))
        a0 = torch.ones(C, D, dtype=torch.float64, device=self.device) if alpha0 is None else \
            torch.as_tensor(np.asarray(alpha0, np.float64) if not torch.is_tensor(alpha0) else alpha0,
                            dtype=torch.float64).to(self.device).contiguous()
        self.ws_bytes = _c.cmtcs_workspace_size(self.problem)
        self.workspace = torch.empty(self.ws_bytes + 256, dtype=torch.uint8, device=self.device)
        ws_ptr = (self.workspace.data_ptr() + 255) & ~255
        self.stream = torch.cuda.current_stream(self.device) if stream is None else stream
        self.ctx = _c.cmtcs_init(self.problem, None if fourier else self.phi.data_ptr(), self.y.data_ptr(), a0.data_ptr(),
                                 ws_ptr, self.ws_bytes, nccl_uid, rank, world,
                                 self.device.index if self.device.index is not None else 0,
                                 self.stream.cuda_stream)
        self.history: list = []

    # ---- Alg. 2 ------------------------------------------------------------------------
    def em_step(self, n_iters: int = 1, probe_bits: torch.Tensor | None = None,
                q_override: torch.Tensor | None = None) -> dict:
        pb = probe_bits.data_ptr() if probe_bits is not None else None
        qo = q_override.data_ptr() if q_override is not None else None
        info = _c.cmtcs_em_step(self.ctx, n_iters, pb, qo)
        self.history.append(info)
        return info

    def fit(self, iters: int) -> dict:
        for _ in range(iters):
            self.em_step(1)
        return self.posterior()

    def posterior(self) -> dict:
        dev, f64 = self.device, torch.float64
        out = dict(mu=torch.empty(self.T_loc, self.C, self.D, dtype=f64, device=dev),
                   s=torch.empty(self.T_loc, self.C, self.D, dtype=f64, device=dev),
                   logdet=torch.empty(self.T_loc, self.C, dtype=f64, device=dev),
                   q=torch.empty(self.T_loc, self.C, dtype=f64, device=dev),
                   alpha=torch.empty(self.C, self.D, dtype=f64, device=dev),
                   assign=torch.empty(self.T_loc, dtype=torch.int32, device=dev),
                   recon=torch.empty(self.T_loc, self.D, dtype=f64, device=dev))
        _c.cmtcs_posterior(self.ctx, *(out[k].data_ptr() for k in ("mu", "s", "logdet", "q", "alpha",
                                                                    "assign", "recon")))
        self.stream.synchronize()
        return out

    def pi(self) -> np.ndarray:
        """The current mixture weights π (learned ones after each M-step when learn_pi)."""
        out = np.zeros(self.C, np.float64)
        _c.cmtcs_get_pi(self.ctx, out.ctypes.data)
        return out

    def set_state(self, alpha, em_iter: int):
        a = torch.as_tensor(np.asarray(alpha, np.float64) if not torch.is_tensor(alpha) else alpha,
                            dtype=torch.float64).to(self.device).contiguous()
        _c.cmtcs_set_state(self.ctx, a.data_ptr(), int(em_iter))
        self.stream.synchronize()

    def transcript(self) -> dict:
        dev = self.device
        cap = self.problem.cg_max_iters
        n = self.T_loc * self.C * self.K
        out = dict(gamma=torch.empty(n, cap, dtype=torch.float64, device=dev),
                   xi=torch.empty(n, cap, dtype=torch.float64, device=dev),
                   steps=torch.empty(n, dtype=torch.int32, device=dev),
                   mu_steps=torch.empty(self.T_loc * self.C, dtype=torch.int32, device=dev))
        _c.cmtcs_transcript(self.ctx, *(out[k].data_ptr() for k in ("gamma", "xi", "steps", "mu_steps")))
        self.stream.synchronize()
        return out

    def estep_sums(self) -> torch.Tensor:
        """This rank's Eq. 4 sums [den (C·D) | num (C) | Σ_t log p(y_t)] before the all-reduce."""
        out = torch.empty(self.C * self.D + self.C + 1, dtype=torch.float64, device=self.device)
        _c.cmtcs_estep_sums(self.ctx, out.data_ptr())
        return out

    def set_timing(self, enable: bool = True):
        _c.cmtcs_set_timing(self.ctx, enable)

    def get_timing(self, reset: bool = False) -> dict:
        return _c.cmtcs_get_timing(self.ctx, reset)

    @property
    def kernel_launches(self) -> int:
        return _c.cmtcs_kernel_launches(self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            _c.cmtcs_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def probe_words(seed: int, it: int, T: int, t0: int, T_loc: int, C: int, K: int, D: int,
                device="cuda") -> torch.Tensor:
    """Probe words of the counter hash (reading A6) computed by the library's kernel."""
    nw = (D + 63) // 64
    out = torch.empty(T_loc * C * K * nw, dtype=torch.int64, device=device)
    _c.cmtcs_probe_words(seed, it, T, t0, T_loc, C, K, D, out.data_ptr(),
                         torch.cuda.current_stream(out.device).cuda_stream)
    torch.cuda.current_stream(out.device).synchronize()
    return out.view(T_loc, C, K, nw)


def lanczos_quadrature(gamma: torch.Tensor, xi: torch.Tensor, steps: torch.Tensor, D: int) -> torch.Tensor:
    """τ_j = D Σ_u S̄²_{u,1} log λ̄_u for every row j (Eq. 7-8), computed by the library's kernel."""
    n, ld = gamma.shape
    gamma = gamma.to(torch.float64).contiguous()
    xi = xi.to(torch.float64).contiguous()
    steps = steps.to(torch.int32).contiguous()
    tau = torch.empty(n, dtype=torch.float64, device=gamma.device)
    scratch = torch.empty(max(1, 3 * n * ld), dtype=torch.float64, device=gamma.device)
    _c.cmtcs_lanczos_quadrature(gamma.data_ptr(), xi.data_ptr(), steps.data_ptr(), n, ld, D, tau.data_ptr(),
                                scratch.data_ptr(), torch.cuda.current_stream(gamma.device).cuda_stream)
    return tau
