"""B200-native CoFEM hot path (arXiv 2310.00420): batched-CG E-step + M-step on sm_100a.

The compute lives in libcmtcs.so (C ABI: include/cmtcs.h; kernels: csrc/).  `cmtcs` is the
ctypes binding with the ABI's names; `model.CoFEM` wraps it with PyTorch-owned device memory.
"""
from .cmtcs import CmtcsError, LIB_PATH  # noqa: F401  (loads libcmtcs.so; raises if missing)
from .model import CoFEM, lanczos_quadrature, probe_words  # noqa: F401
