"""ctypes binding of libfeastb200.so (the C ABI in include/feast_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every device entry point raises ``FeastB200Unavailable``.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfeastb200.so")

c_int, c_int64, c_double, c_char, c_void_p, c_size_t, c_uint64 = (
    ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_char, ctypes.c_void_p,
    ctypes.c_size_t, ctypes.c_uint64)
P = c_void_p
PI = ctypes.POINTER(c_int)

# name -> (restype, argtypes); mirrors include/feast_b200.h exactly
SIGNATURES = {
    "fb_abi_version": (c_int, []),
    "fb_ctx_create": (c_int, [c_int, P, ctypes.POINTER(P)]),
    "fb_ctx_destroy": (c_int, [P]),
    "fb_ctx_set_stream": (c_int, [P, P]),
    "fb_ctx_synchronize": (c_int, [P]),
    "fb_ctx_last_error": (ctypes.c_char_p, [P]),
    "fb_ctx_launch_count": (c_int64, [P]),
    "fb_dense_shift": (c_int, [P, c_int, c_double, c_double, P, P, c_int64, P, P, c_int64, P, P, c_int64]),
    "fb_zgetrf_dinv_doubles": (c_size_t, [c_int]),
    "fb_zgetrf": (c_int, [P, c_int, P, P, c_int64, P, P, P]),
    "fb_read_info": (c_int, [P, P, PI]),
    "fb_zgetrs": (c_int, [P, c_int, c_int, P, P, c_int64, P, P, c_int, P, P, c_int64]),
    "fb_dense_shift_batched": (c_int, [P, c_int, c_int, P, P, P, P, c_int64, P, P, c_int64, P, P, c_int64,
                                       c_int64]),
    "fb_zgetrf_batched": (c_int, [P, c_int, c_int, P, P, c_int64, c_int64, P, c_int64, P, c_int64, P]),
    "fb_read_info_batched": (c_int, [P, c_int, P, P]),
    "fb_zgetrs_batched": (c_int, [P, c_int, c_int, c_int, P, P, c_int64, c_int64, P, c_int64, P, c_int64,
                                  c_int, P, P, c_int64, c_int64, P, P, c_int64, c_int64]),
    "fb_splitmix": (c_int, [P, c_uint64, c_int64, c_int64, c_int, c_int, P, P, c_int64]),
    "fb_accumulate": (c_int, [P, c_int, c_int, c_int, P, P, c_int64, P, P, c_int64, c_double,
                              c_double, c_double]),
    "fb_accumulate_terms": (c_int, [P, c_int, P, P, c_double, P, P, P, c_int, c_int, c_int64, P, P, c_int64]),
    "fb_gemm": (c_int, [P, c_int, c_char, c_char, c_int, c_int, c_int, c_double, c_double, P, P,
                        c_int64, P, P, c_int64, c_double, c_double, P, P, c_int64]),
    "fb_symmetrize": (c_int, [P, c_int, P, P, c_int64]),
    "fb_residuals": (c_int, [P, c_int, c_int, P, P, P, P, c_int64, P, c_double, P]),
    "fb_residual_sums": (c_int, [P, c_int, c_int, P, P, P, P, c_int64, P, c_double, P]),
    "fb_chol_check": (c_int, [P, c_int, P, P, c_int64, PI]),
    "fb_reduced_eig": (c_int, [P, c_int, P, P, P, P, c_int64, P, P, P, c_int64, PI]),
    "fb_pack": (c_int, [P, c_int, c_int, P, c_int64, P, P, c_int64, c_int]),
    "fb_band_matvec": (c_int, [P, c_int, c_int, c_int, P, P, c_int64, P, P, c_int64, P, P, c_int64]),
    "fb_band_factor": (c_int, [P, c_int, c_int, c_double, c_double, P, P, P, P, c_int64, P, P, P, P]),
    "fb_band_solve": (c_int, [P, c_int, c_int, c_int, P, P, P, c_int, P, P, c_int64]),
    "fb_band_aux_doubles": (c_int64, [c_int, c_int]),
    "fb_band_factor_batched": (c_int, [P, c_int, c_int, c_int, P, P, P, P, P, P, c_int64, P, P, c_int64,
                                       P, c_int64, P, c_int64, P]),
    "fb_band_solve_batched_rhs": (c_int, [P, c_int, c_int, c_int, c_int, P, P, c_int64, P, c_int64, P, c_int64,
                                          P, P, c_int64, c_int64, P, P, c_int64, c_int64]),
    "fb_band_solve_accumulate": (c_int, [P, c_int, c_int, c_int, c_int, P, P, c_int64, P, c_int64, P, c_int64,
                                         P, P, c_int64, P, P, c_int64, c_int64, c_int, P, P, P, c_double, P,
                                         P, P, c_int64]),
    "fb_band_solve_batched": (c_int, [P, c_int, c_int, c_int, c_int, P, P, c_int64, P, c_int64, P, c_int64,
                                      P, P, c_int64, c_int64]),
    "fb_csr_matvec": (c_int, [P, c_int, c_int, P, P, P, P, P, P, c_int64, P, P, c_int64, P]),
    "fb_permute_rows": (c_int, [P, c_int, c_int, P, P, P, c_int64, P, P, c_int64]),
    "fb_bicgstab_workspace_doubles": (c_int64, [c_int, c_int, c_int64]),
    "fb_bicgstab": (c_int, [P, c_int, c_int, c_int, P, P, P, P, P, P, P, P, c_int64, P, P, c_int64, c_double,
                            c_int, c_int, P, c_int64, P, P]),
}

FB_OK, FB_ERR_ALLOC, FB_ERR_SINGULAR, FB_ERR_REDUCED, FB_ERR_ARG, FB_ERR_CUDA = 0, -1, -2, -3, -10, -11


class FeastB200Unavailable(RuntimeError):
    """libfeastb200.so is missing, stale, or no CUDA device is present."""


_lib = None


def load(path: str = LIB_PATH):
    """Load and bind the shared library (no compute; safe without a GPU)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FeastB200Unavailable(
            f"{path} not found: build it with `python -m paper_1203_4031_b200.build` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.fb_abi_version() != 1:
        raise FeastB200Unavailable("libfeastb200.so ABI mismatch")
    _lib = lib
    return lib
