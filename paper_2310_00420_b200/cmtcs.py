"""Thin ctypes binding of libcmtcs.so (include/cmtcs.h), same names as the C ABI.

Argument marshalling only: every step of the CoFEM path runs in the library's sm_100a kernels.
PyTorch is used for device memory (tensors whose data pointers are passed through) and streams.
There is no CPU fallback: if the shared library is missing, importing the bindings raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, byref, c_char_p, c_double, c_int32, c_int64, c_size_t, c_uint8, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcmtcs.so")

STATUS = {0: "CMTCS_OK", 1: "CMTCS_EINVAL", 2: "CMTCS_ENOMEM", 3: "CMTCS_ECUDA", 4: "CMTCS_ENCCL",
          5: "CMTCS_EBREAKDOWN", 6: "CMTCS_EEIG", 7: "CMTCS_ENUMERIC", 8: "CMTCS_ESTATE"}

EXPORTED = ["cmtcs_get_unique_id", "cmtcs_workspace_size", "cmtcs_init", "cmtcs_em_step",
            "cmtcs_posterior", "cmtcs_set_state", "cmtcs_transcript", "cmtcs_last_error",
            "cmtcs_destroy", "cmtcs_kernel_launches", "cmtcs_probe_words", "cmtcs_lanczos_quadrature",
            "cmtcs_set_timing", "cmtcs_get_timing", "cmtcs_estep_sums", "cmtcs_get_pi"]


class CmtcsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class cmtcs_problem(ctypes.Structure):
    _fields_ = [("T", c_int32), ("N", c_int32), ("D", c_int32), ("C", c_int32), ("K", c_int32),
                ("shared_phi", c_int32), ("beta", c_double), ("pi", POINTER(c_double)),
                ("cg_max_iters", c_int32), ("cg_rel_tol", c_double), ("alpha_max", c_double),
                ("var_floor", c_double), ("empty_eps", c_double), ("probe_seed", c_uint64),
                ("task_begin", c_int32), ("task_end", c_int32), ("em_iter0", c_int32),
                ("mean_rel_tol", c_double), ("op_kind", c_int32), ("fourier_rows", c_void_p),
                ("learn_pi", c_int32)]


CMTCS_OP_DENSE, CMTCS_OP_PARTIAL_FOURIER, CMTCS_OP_DENSE_FP32 = 0, 1, 2


class cmtcs_step_info(ctypes.Structure):
    _fields_ = [("loglik", c_double), ("em_iter", c_int32), ("cg_iters", c_int32),
                ("mu_steps_min", c_int32), ("mu_steps_max", c_int32),
                ("probe_steps_min", c_int32), ("probe_steps_max", c_int32),
                ("probe_steps_mean", c_double), ("n_cap_hit", c_int64),
                ("probe_col_iters", c_int64), ("mean_col_iters", c_int64),
                ("task_iters", c_int64), ("kernel_launches", c_int64), ("tile_col_iters", c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python __graft_entry__.py` (build()) first")
    lib = ctypes.CDLL(LIB_PATH)
    st = c_int32
    vp = c_void_p
    lib.cmtcs_get_unique_id.argtypes = [POINTER(c_uint8)]
    lib.cmtcs_get_unique_id.restype = st
    lib.cmtcs_workspace_size.argtypes = [POINTER(cmtcs_problem), POINTER(c_size_t)]
    lib.cmtcs_workspace_size.restype = st
    lib.cmtcs_init.argtypes = [POINTER(vp), POINTER(cmtcs_problem), vp, vp, vp, vp, c_size_t,
                               POINTER(c_uint8), c_int32, c_int32, c_int32, vp]
    lib.cmtcs_init.restype = st
    lib.cmtcs_em_step.argtypes = [vp, c_int32, vp, vp, POINTER(cmtcs_step_info)]
    lib.cmtcs_em_step.restype = st
    lib.cmtcs_posterior.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp]
    lib.cmtcs_posterior.restype = st
    lib.cmtcs_set_state.argtypes = [vp, vp, c_int32]
    lib.cmtcs_set_state.restype = st
    lib.cmtcs_transcript.argtypes = [vp, vp, vp, vp, vp]
    lib.cmtcs_transcript.restype = st
    lib.cmtcs_last_error.argtypes = [vp]
    lib.cmtcs_last_error.restype = c_char_p
    lib.cmtcs_destroy.argtypes = [vp]
    lib.cmtcs_destroy.restype = None
    lib.cmtcs_kernel_launches.argtypes = [vp]
    lib.cmtcs_kernel_launches.restype = c_int64
    lib.cmtcs_probe_words.argtypes = [c_uint64, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32,
                                      c_int32, vp, vp]
    lib.cmtcs_probe_words.restype = st
    lib.cmtcs_lanczos_quadrature.argtypes = [vp, vp, vp, c_int32, c_int32, c_int32, vp, vp, vp]
    lib.cmtcs_lanczos_quadrature.restype = st
    lib.cmtcs_set_timing.argtypes = [vp, c_int32]
    lib.cmtcs_set_timing.restype = st
    lib.cmtcs_get_timing.argtypes = [vp, POINTER(c_double), POINTER(c_int64), c_int32]
    lib.cmtcs_get_timing.restype = st
    lib.cmtcs_estep_sums.argtypes = [vp, vp]
    lib.cmtcs_estep_sums.restype = st
    lib.cmtcs_get_pi.argtypes = [vp, vp]
    lib.cmtcs_get_pi.restype = st
    return lib


_lib = _load()


def _check(status: int, ctx=None):
    if status != 0:
        msg = _lib.cmtcs_last_error(ctx)
        raise CmtcsError(status, msg.decode() if msg else "")


# ---- same-name wrappers -------------------------------------------------------------------
def cmtcs_get_unique_id() -> bytes:
    buf = (c_uint8 * 128)()
    _check(_lib.cmtcs_get_unique_id(buf))
    return bytes(buf)


def cmtcs_workspace_size(problem: cmtcs_problem) -> int:
    n = c_size_t(0)
    _check(_lib.cmtcs_workspace_size(byref(problem), byref(n)))
    return n.value


def cmtcs_init(problem: cmtcs_problem, phi_ptr: int, y_ptr: int, alpha0_ptr: int, ws_ptr: int,
               ws_bytes: int, nccl_uid: bytes | None, rank: int, world: int, device: int,
               stream: int) -> int:
    ctx = c_void_p()
    uid = (c_uint8 * 128).from_buffer_copy(nccl_uid) if nccl_uid else None
    st = _lib.cmtcs_init(byref(ctx), byref(problem), phi_ptr, y_ptr, alpha0_ptr, ws_ptr, ws_bytes,
                         uid, rank, world, device, stream)
    if st != 0:
        msg = _lib.cmtcs_last_error(ctx if ctx.value else None)
        if ctx.value:
            _lib.cmtcs_destroy(ctx)
        raise CmtcsError(st, msg.decode() if msg else "")
    return ctx.value


def cmtcs_em_step(ctx: int, n_iters: int = 1, probe_bits_ptr: int | None = None,
                  q_override_ptr: int | None = None) -> dict:
    info = cmtcs_step_info()
    _check(_lib.cmtcs_em_step(ctx, n_iters, probe_bits_ptr, q_override_ptr, byref(info)), ctx)
    return info.as_dict()


def cmtcs_posterior(ctx: int, mu=None, s=None, logdet=None, q=None, alpha=None, assign=None, recon=None):
    _check(_lib.cmtcs_posterior(ctx, mu, s, logdet, q, alpha, assign, recon), ctx)


def cmtcs_set_state(ctx: int, alpha_ptr: int | None, em_iter: int):
    _check(_lib.cmtcs_set_state(ctx, alpha_ptr, em_iter), ctx)


def cmtcs_transcript(ctx: int, gamma=None, xi=None, steps=None, mu_steps=None):
    _check(_lib.cmtcs_transcript(ctx, gamma, xi, steps, mu_steps), ctx)


def cmtcs_last_error(ctx: int | None) -> str:
    m = _lib.cmtcs_last_error(ctx)
    return m.decode() if m else ""


def cmtcs_destroy(ctx: int):
    _lib.cmtcs_destroy(ctx)


def cmtcs_kernel_launches(ctx: int) -> int:
    return int(_lib.cmtcs_kernel_launches(ctx))


def cmtcs_probe_words(seed: int, it: int, T: int, t0: int, T_loc: int, C: int, K: int, D: int,
                      out_ptr: int, stream: int = 0):
    _check(_lib.cmtcs_probe_words(seed, it, T, t0, T_loc, C, K, D, out_ptr, stream))


def cmtcs_lanczos_quadrature(gamma_ptr: int, xi_ptr: int, steps_ptr: int, n: int, ld: int, D: int,
                             tau_ptr: int, scratch_ptr: int, stream: int = 0):
    _check(_lib.cmtcs_lanczos_quadrature(gamma_ptr, xi_ptr, steps_ptr, n, ld, D, tau_ptr, scratch_ptr,
                                         stream))


def cmtcs_set_timing(ctx: int, enable: bool):
    _check(_lib.cmtcs_set_timing(ctx, 1 if enable else 0), ctx)


def cmtcs_get_timing(ctx: int, reset: bool = False) -> dict:
    ms = (c_double * 4)()
    n = (c_int64 * 4)()
    _check(_lib.cmtcs_get_timing(ctx, ms, n, 1 if reset else 0), ctx)
    return dict(op_ms=ms[0], update_ms=ms[1], other_ms=ms[2], cg_kernel_ms=ms[3], op_steps=n[0],
                update_steps=n[1], em_iters=n[2], cg_kernel_launches=n[3])


def cmtcs_estep_sums(ctx: int, out_ptr: int):
    _check(_lib.cmtcs_estep_sums(ctx, out_ptr), ctx)


def cmtcs_get_pi(ctx: int, out_ptr: int):
    _check(_lib.cmtcs_get_pi(ctx, out_ptr), ctx)
