"""The SRM subset of the reference's dense kernels, on the device.

Drop-in for the four functions of ``factorfit.kernels`` that the SRM path
calls (``/root/reference/pkg/src/factorfit/kernels.py:39-47, 152-212``):
same names, argument meanings, return types (numpy arrays / floats) and
exceptions.  Every piece of arithmetic runs in libsrm_b200.so; there is no
CPU fallback.

* ``trace_ata``        -> ``srm_trace_ata`` (fixed-order sum of squares)
* ``add_diag``         -> ``srm_add_diag``
* ``spd_inverse``      -> ``srm_spd_inverse`` (register Cholesky/LDL^T sweep;
  ``DefinitenessError.pivot`` is the 0-based dpotrf pivot)
* ``polar_orthogonal`` -> ``srm_polar`` (Householder TSQR + one-sided Jacobi
  SVD of R; ``RankError`` when sigma_min < 1e-12 sigma_max)

The reference's ``_as_matrix`` guard (kernels.py:39-47) is kept: 2-D with at
least one row and column (``ShapeError``), finite entries
(``InvalidInputError``, checked on the device by the sum-of-squares kernel).
"""

import numpy as np

from . import _lib
from .errors import ShapeError

__all__ = ["trace_ata", "add_diag", "spd_inverse", "polar_orthogonal", "RANK_TOLERANCE"]

#: kernels.py:31-33 -- the polar rank threshold (sigma_min / sigma_max)
RANK_TOLERANCE = 1e-12


def _srm():
    from . import srm

    return srm


def _matrix(a, name="A"):
    """Host-side shape part of kernels.py:39-47 -> contiguous fp64 CUDA tensor."""
    srm = _srm()
    torch = srm._torch()
    arr = a if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ShapeError(f"{name} must be 2-D, got ndim={arr.ndim}")
    if arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ShapeError(f"{name} must have at least one row and column")
    return srm._dev(arr, torch.float64)


def _sumsq(dev):
    """(device scalar tensor, status) of the fixed-order sum of squares."""
    srm = _srm()
    torch = srm._torch()
    lib = _lib.load()
    out = torch.empty(1, dtype=torch.float64, device=dev.device)
    ws = torch.empty(1024, dtype=torch.float64, device=dev.device)
    st = srm._status_tensor()
    _lib.check(lib.srm_trace_ata(srm._ptr(dev), srm._ld(dev), dev.shape[0], dev.shape[1], srm._ptr(out),
                                 srm._ptr(st), srm._ptr(ws), ws.numel() * 8, srm._stream()), "trace_ata")
    return out, st


def _check_finite(dev):
    _, st = _sumsq(dev)
    _srm()._raise_status(st)


def trace_ata(A):
    """trace(A^T A) as the sum of squared entries (kernels.py:152-155)."""
    dev = _matrix(A)
    out, st = _sumsq(dev)
    _srm()._raise_status(st)
    return float(out.item())


def add_diag(A, c):
    """A + c I; off-diagonal entries untouched (kernels.py:158-165)."""
    srm = _srm()
    torch = srm._torch()
    dev = _matrix(A)
    if dev.shape[0] != dev.shape[1]:
        raise ShapeError(f"add_diag needs a square matrix, got {tuple(dev.shape)}")
    _check_finite(dev)
    n = dev.shape[0]
    out = torch.empty((n, n), dtype=torch.float64, device=dev.device)
    _lib.check(_lib.load().srm_add_diag(srm._ptr(dev), srm._ld(dev), n, float(c), srm._ptr(out), n,
                                        srm._stream()), "add_diag")
    return out.cpu().numpy()


def spd_inverse(A):
    """Inverse of a symmetric positive definite matrix (kernels.py:168-187).

    ``DefinitenessError(pivot)`` names the 0-based pivot at which the
    Cholesky factorisation breaks down, as dpotrf's ``info - 1``.
    """
    srm = _srm()
    torch = srm._torch()
    dev = _matrix(A)
    if dev.shape[0] != dev.shape[1]:
        raise ShapeError(f"spd_inverse needs a square matrix, got {tuple(dev.shape)}")
    _check_finite(dev)
    n = dev.shape[0]
    work = dev.clone()
    st = srm._status_tensor()
    _lib.check(_lib.load().srm_spd_inverse(srm._ptr(work), n, srm._ptr(st), srm._stream()), "spd_inverse")
    srm._raise_status(st)
    return work.cpu().numpy()


def polar_orthogonal(A):
    """Orthogonal polar factor W = U V^T of A (kernels.py:190-212).

    ``ShapeError`` when rows < cols, ``RankError`` when the smallest singular
    value is below ``RANK_TOLERANCE`` times the largest.
    """
    srm = _srm()
    dev = _matrix(A)
    rows, cols = dev.shape
    if rows < cols:
        raise ShapeError(f"polar_orthogonal needs rows >= cols, got {tuple(dev.shape)}")
    _check_finite(dev)
    return srm._polar(dev, cols).cpu().numpy()
