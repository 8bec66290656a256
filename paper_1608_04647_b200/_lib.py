"""ctypes binding of the C ABI in ``include/srm_b200.h`` (libsrm_b200.so).

The library is built in-tree (``make`` / ``__graft_entry__.build()``) for
sm_100a.  There is no fallback: if the shared object is missing or a call
fails, the caller gets an exception.
"""

import ctypes
import os
from pathlib import Path

from .errors import DeviceError, from_status

LIB_PATH = Path(__file__).resolve().parent / "libsrm_b200.so"

c_int = ctypes.c_int
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_i64p = ctypes.POINTER(ctypes.c_int64)

# (name, restype, argtypes) for every symbol declared in include/srm_b200.h
SIGNATURES = [
    ("srm_abi_version", c_int, []),
    ("srm_last_error", ctypes.c_char_p, []),
    ("srm_plan_create", c_int, [ctypes.POINTER(c_vp), c_int, c_int, c_i64p, c_i64, c_i64, c_int,
                                c_int, c_int, c_i32p, c_int]),
    ("srm_plan_destroy", c_int, [c_vp]),
    ("srm_plan_workspace_bytes", c_i64, [c_vp]),
    ("srm_plan_dim", c_i64, [c_vp, c_int]),
    ("srm_plan_bind", c_int, [c_vp, c_vp, c_i64]),
    ("srm_plan_region", c_int, [c_vp, c_int, c_i64p, c_i64p]),
    ("srm_load_subject", c_int, [c_vp, c_int, c_vp, c_int, c_i64, c_vp]),
    ("srm_finish_load", c_int, [c_vp, c_vp]),
    ("srm_init_mapping", c_int, [c_vp, c_vp]),
    ("srm_init_mapping_range", c_int, [c_vp, c_int, c_int, c_vp]),
    ("srm_prepare_gram", c_int, [c_vp, c_vp]),
    ("srm_prepare_gram_range", c_int, [c_vp, c_int, c_int, c_vp]),
    ("srm_reset", c_int, [c_vp, c_vp]),
    ("srm_set_iteration", c_int, [c_vp, c_int, c_vp]),
    ("srm_reduce_local", c_int, [c_vp, c_vp]),
    ("srm_xchg_pack", c_int, [c_vp, c_vp]),
    ("srm_xchg_reduce", c_int, [c_vp, c_vp]),
    ("srm_xchg_unpack", c_int, [c_vp, c_vp]),
    ("srm_e_step", c_int, [c_vp, c_vp]),
    ("srm_m_step", c_int, [c_vp, c_vp]),
    ("srm_finalize", c_int, [c_vp, c_vp]),
    ("srm_finalize_range", c_int, [c_vp, c_int, c_int, c_vp]),
    ("srm_graph_capture", c_int, [c_vp]),
    ("srm_graph_launch", c_int, [c_vp, c_vp]),
    ("srm_profile_iteration", c_int, [c_vp, ctypes.POINTER(ctypes.c_float), c_int, c_i32p, c_vp]),
    ("srm_profile_gram", c_int, [c_vp, ctypes.POINTER(ctypes.c_float), c_int, c_i32p, c_vp]),
    ("srm_profile_finalize", c_int, [c_vp, ctypes.POINTER(ctypes.c_float), c_int, c_i32p, c_vp]),
    ("srm_profile_name", ctypes.c_char_p, [c_int]),
    ("srm_read_status", c_int, [c_vp, c_i32p]),
    ("srm_clear_status", c_int, [c_vp, c_vp]),
    ("srm_gemm_tn", c_int, [c_vp, c_i64, c_vp, c_int, c_i64, c_i64, c_i64, c_i64, c_dbl, c_vp,
                            c_i64, c_vp, c_i64, c_vp]),
    ("srm_gemm_nt", c_int, [c_vp, c_int, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_dbl, c_vp,
                            c_i64, c_vp, c_i64, c_vp]),
    ("srm_tail_step", c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_dbl, c_vp, c_i64, c_vp,
                              c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    ("srm_project", c_int, [c_vp, c_i64, c_vp, c_int, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp,
                            c_i64, c_vp]),
    ("srm_unproject", c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp]),
    ("srm_trace_ata", c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp]),
    ("srm_add_diag", c_int, [c_vp, c_i64, c_i64, c_dbl, c_vp, c_i64, c_vp]),
    ("srm_dot", c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp]),
    ("srm_sigma_update", c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp]),
    ("srm_spd_inverse", c_int, [c_vp, c_i64, c_vp, c_vp]),
    ("srm_polar", c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp]),
    ("srm_stateless_workspace_bytes", c_i64, [c_i64, c_i64, c_i64]),
    ("srm_sfab_header", c_int, [ctypes.c_char_p, c_i64p, c_i64p]),
    ("srm_sfab_read", c_int, [ctypes.c_char_p, c_vp, c_i64, c_int]),
    ("srm_sfab_write", c_int, [ctypes.c_char_p, ctypes.POINTER(c_dbl), c_i64, c_i64]),
    ("srm_sfab_last_error", ctypes.c_char_p, [c_i64p, ctypes.POINTER(ctypes.c_char_p)]),
]

# include/srm_b200.h enums
SRM_F64, SRM_F32 = 0, 1
FLAG_ORDERED, FLAG_TOLERANCE, FLAG_GRAM, FLAG_TC, FLAG_GRAM_I8, FLAG_EXACT_POLAR, FLAG_COLBLOCK = 1, 2, 4, 8, 16, 32, 64
WARN_POLAR_CONDITION = 1
(R_XHAT, R_AMAT, R_WOUT, R_MU, R_TERMS, R_RED, R_REDLOCAL, R_S, R_SIGMA, R_HIST, R_STATUS,
 R_MMAT, R_SCAL, R_GRAM, R_VAR, R_XSEND, R_XRECV, R_XRED) = range(18)
(D_LDX, D_KP, D_ROWS, D_TERM_STRIDE, D_RED_STRIDE, D_HIST_STRIDE, D_N_SLOTS, D_SLOT_OFFSET,
 D_ITEMS_E, D_ITEMS_A, D_CHUNK_ROWS, D_LAUNCHES, D_FLAGS, D_XREC, D_XRED) = range(15)
H_LL, H_TRACE, H_RHO0, H_SDIFF, H_SPREV, H_RHO2 = 0, 1, 2, 3, 4, 8
REC_RHO2, REC_V, REC_SQNORM, REC_SCALARS = 0, 1, 2, 8
RED_RHO0, RED_VLOGRHO, RED_SQRHO, RED_VSUM = 0, 1, 2, 3

_LIB = None


def load():
    """Load libsrm_b200.so once; raise DeviceError if it is not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = Path(os.environ.get("SRM_B200_LIB", LIB_PATH))
    if not path.exists():
        raise DeviceError(
            f"{path} is missing: build the CUDA library first (`make` at the repo root "
            "or `python -c 'import __graft_entry__ as g; g.build()'`); there is no CPU fallback"
        )
    lib = ctypes.CDLL(str(path))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.srm_abi_version() != 1:
        raise DeviceError("libsrm_b200.so ABI version mismatch")
    _LIB = lib
    return lib


def check_sfab(code):
    """Raise the reference's exception for a failed srm_sfab_* call."""
    if code != 0:
        off = c_i64()
        field = ctypes.c_char_p()
        msg = _LIB.srm_sfab_last_error(ctypes.byref(off), ctypes.byref(field)).decode()
        fld = field.value.decode() if field.value else None
        raise from_status(code, msg, offset=off.value if off.value >= 0 else None, field=fld)


def check(code, what=""):
    """Raise the mapped exception for a non-zero status return."""
    if code != 0:
        msg = _LIB.srm_last_error().decode() if _LIB is not None else ""
        raise from_status(code, f"{what}: {msg}" if what else msg)
