"""Shared response model fit on B200: the reference ``factorfit.srm`` API.

Drop-in for ``/root/reference/pkg/src/factorfit/srm.py``: the same names
(``__all__``), argument meanings, return types and exceptions.  Every piece
of arithmetic runs in hand-written sm_100a CUDA (libsrm_b200.so, fp64 on
the FP64 tensor cores); Python only orchestrates, as the reference's
``fit`` does.  There is no CPU fallback -- without the library or a GPU the
calls raise.

The EM iteration (srm.py:254-287) on the device:

* E-step term ``W_i^T Xhat_i / rho_i^2`` is never formed from ``W_i``:
  with ``A_i = Xhat_i S^T / 2`` and ``M_i = (A_i^T A_i)^{-1/2}`` the polar
  factor is ``W_i = A_i M_i`` (kernels.py:190-212, unique for full rank), so
  ``W_i^T Xhat_i = M_i^T (A_i^T Xhat_i)``.  One product serves both the
  M-step cross term (srm.py:151) and the next E-step (srm.py:118); ``W_i``
  is materialised once at the end.
* the reduction sums the per-subject terms in ascending global subject
  order (srm.py:193-213) from an all-gathered table, so ``S`` is identical
  on every rank and for every shard layout.
* the K x K algebra (two Cholesky inverses, S, Sigma_s, trace) runs
  redundantly on every rank: no broadcast (srm.py:266-269) is needed.
"""

import ctypes
import os
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib, hostio
from .collectives import SerialCommunicator, TorchCommunicator, any_rank, rank_counts
from .data import SubjectData
from .engine import SrmEngine, reference_gaussian
from .errors import ConfigError, DeviceError, ShapeError, from_status

__all__ = [
    "SrmConfig",
    "SrmModel",
    "SubjectData",
    "demean",
    "init_subject",
    "e_step_local",
    "e_step_global",
    "update_sigma_s",
    "m_step_subject",
    "fit",
    "project",
    "map_between",
    "project_batch",
    "map_between_batch",
    "IterationState",
]

RHO_FLOOR = 1e-12


@dataclass
class SrmConfig:
    """srm.py:54-67."""

    k: int
    iterations: int = 10
    seed: int = 0
    tolerance: Optional[float] = None

    def validate(self):
        if self.k < 1:
            raise ConfigError("k must be at least 1")
        if self.iterations < 1:
            raise ConfigError("iterations must be at least 1")
        if self.tolerance is not None and self.tolerance <= 0:
            raise ConfigError("tolerance must be positive when given")


@dataclass
class SrmModel:
    """Fitted model state held by one worker (srm.py:70-91).

    Extra fields beyond the reference: ``log_likelihood`` (per iteration,
    the marginal log-likelihood of the parameters that entered that
    iteration's E-step) and ``device_state`` (the engine, when the caller
    asked to keep results on the GPU).
    """

    subject_ids: list
    subject_indices: list
    W: list
    rho2: list
    mu: list
    S: np.ndarray
    rho0: float
    n_subjects: int
    sigma_s: Optional[np.ndarray] = None
    rho2_all: Optional[np.ndarray] = None
    objective_trace: list = field(default_factory=list)
    log_likelihood: list = field(default_factory=list)
    device_state: object = None


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

def _torch():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("a CUDA device is required (no CPU fallback)")
    return torch


def _dev(a, dtype=None):
    """Host/device array -> contiguous float64 (or float32) CUDA tensor."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        t = a.detach()
        if dtype is None:
            dtype = t.dtype if t.dtype in (torch.float64, torch.float32) else torch.float64
        return t.to(device="cuda", dtype=dtype).contiguous()
    arr = np.asarray(a)
    if dtype is None:
        dtype = torch.float32 if arr.dtype == np.float32 else torch.float64
    np_dt = np.float32 if dtype == torch.float32 else np.float64
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np_dt)).to("cuda")


def _as_matrix(a, name="matrix"):
    arr = a if hasattr(a, "shape") else np.asarray(a)
    if len(arr.shape) != 2:
        raise ShapeError(f"{name} must be 2-D, got ndim={len(arr.shape)}")
    if arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ShapeError(f"{name} must have at least one row and column")
    return arr


def _status_tensor():
    torch = _torch()
    return torch.zeros(4, dtype=torch.int32, device="cuda")


def _raise_status(status):
    code, arg = (int(x) for x in status[:2].tolist())
    if code:
        raise from_status(code, arg=arg)


def _workspace(v, k, t):
    torch = _torch()
    lib = _lib.load()
    nb = int(lib.srm_stateless_workspace_bytes(int(v), int(k), int(t)))
    return torch.empty(nb, dtype=torch.uint8, device="cuda"), nb


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _ld(t):
    """Row pitch in elements of a row-major 2-D tensor (size-1 rows may carry any stride)."""
    return int(t.stride(0)) if t.shape[0] > 1 else int(t.shape[1])


def _stream():
    return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)


def _finite(t, name):
    """kernels.py:45-46 on the device: the sum-of-squares kernel flags
    non-finite entries (InvalidInputError)."""
    torch = _torch()
    lib = _lib.load()
    d = t if t.dtype == torch.float64 else t.to(torch.float64)
    d = d.reshape(d.shape[0], -1) if d.dim() != 2 else d
    out = torch.empty(1, dtype=torch.float64, device=d.device)
    ws = torch.empty(1024, dtype=torch.float64, device=d.device)
    st = _status_tensor()
    _lib.check(lib.srm_trace_ata(_ptr(d), _ld(d), d.shape[0], d.shape[1], _ptr(out), _ptr(st), _ptr(ws), 8192,
                                 _stream()), "finite check")
    if int(st[0].item()):
        from .errors import InvalidInputError

        raise InvalidInputError(f"{name} contains non-finite entries")


# ---------------------------------------------------------------------------
# step functions (srm.py:94-155)
# ---------------------------------------------------------------------------

def demean(X):
    """Remove each voxel's temporal mean; returns (Xhat, mu)  (srm.py:94-98)."""
    torch = _torch()
    x = _as_matrix(X, "X")
    v, t = int(x.shape[0]), int(x.shape[1])
    eng = SrmEngine([v], t, 1, 1, storage="f64")
    try:
        eng.load([x])
    except Exception:
        eng.close()
        raise
    xhat = eng.xhat[:, :t].clone()
    mu = eng.mu[:v].clone()
    eng.close()
    torch.cuda.synchronize()
    return xhat.cpu().numpy(), mu.cpu().numpy()


def _polar(a_dev, k):
    torch = _torch()
    lib = _lib.load()
    v = a_dev.shape[0]
    if v < k:
        raise ShapeError(f"polar_orthogonal needs rows >= cols, got {tuple(a_dev.shape)}")
    ws, nb = _workspace(v, k, 32)
    w = torch.empty((v, k), dtype=torch.float64, device="cuda")
    st = _status_tensor()
    _lib.check(lib.srm_polar(_ptr(a_dev), _ld(a_dev), v, k, _ptr(w), k, _ptr(st), _ptr(ws), nb,
                             _stream()), "polar")
    _raise_status(st)
    return w


def init_subject(n_voxels, config, subject_index):
    """Seeded random orthogonal mapping and unit noise variance (srm.py:101-113)."""
    if n_voxels < config.k:
        raise ShapeError(f"subject has {n_voxels} voxels, fewer than k={config.k} factors")
    g = reference_gaussian(n_voxels, config.k, config.seed, subject_index)
    return _polar(_dev(g), config.k).cpu().numpy(), 1.0


def _gemm_tn(w_dev, x_dev, alpha=1.0):
    torch = _torch()
    lib = _lib.load()
    v, k = w_dev.shape
    t = x_dev.shape[1]
    out = torch.empty((k, t), dtype=torch.float64, device="cuda")
    ws, nb = _workspace(v, k, t)
    dt = _lib.SRM_F64 if x_dev.dtype == torch.float64 else _lib.SRM_F32
    _lib.check(lib.srm_gemm_tn(_ptr(w_dev), _ld(w_dev), _ptr(x_dev), dt, _ld(x_dev), v, k, t,
                               float(alpha), _ptr(out), t, _ptr(ws), nb, _stream()), "gemm_tn")
    return out


def _gemm_nt(x_dev, s_dev, alpha=1.0):
    torch = _torch()
    lib = _lib.load()
    v, t = x_dev.shape
    k = s_dev.shape[0]
    out = torch.empty((v, k), dtype=torch.float64, device="cuda")
    ws, nb = _workspace(v, k, t)
    dt = _lib.SRM_F64 if x_dev.dtype == torch.float64 else _lib.SRM_F32
    _lib.check(lib.srm_gemm_nt(_ptr(x_dev), dt, _ld(x_dev), _ptr(s_dev), _ld(s_dev), v, t, k,
                               float(alpha), _ptr(out), k, _ptr(ws), nb, _stream()), "gemm_nt")
    return out


def e_step_local(W_i, rho2_i, Xhat_i):
    """This subject's term of the reduction: rho_i^{-2} W_i^T Xhat_i (srm.py:116-118)."""
    w = _dev(_as_matrix(W_i, "W"), _torch().float64)
    x = _dev(_as_matrix(Xhat_i, "Xhat"))
    return (_gemm_tn(w, x) / rho2_i).cpu().numpy()


def _tail(reduced, sigma_s, rho0):
    torch = _torch()
    lib = _lib.load()
    red = _dev(_as_matrix(reduced, "reduced"), torch.float64)
    sig = _dev(_as_matrix(sigma_s, "sigma_s"), torch.float64)
    k, t = red.shape
    if sig.shape != (k, k):
        raise ShapeError(f"sigma_s must be {k} x {k}")
    _finite(sig, "A")
    s = torch.empty((k, t), dtype=torch.float64, device="cuda")
    var = torch.empty((k, k), dtype=torch.float64, device="cuda")
    sig_new = torch.empty((k, k), dtype=torch.float64, device="cuda")
    trace = torch.empty(1, dtype=torch.float64, device="cuda")
    ws, nb = _workspace(1, k, t)
    st = _status_tensor()
    _lib.check(lib.srm_tail_step(_ptr(red), t, _ptr(sig), k, k, t, float(rho0), _ptr(s), t, _ptr(var),
                                 _ptr(sig_new), _ptr(trace), _ptr(st), _ptr(ws), nb, _stream()), "tail")
    _raise_status(st)
    return s, var, sig_new, trace


def e_step_global(reduced, sigma_s, rho0):
    """Posterior mean S and covariance from the reduction (srm.py:121-129)."""
    s, var, _, _ = _tail(reduced, sigma_s, rho0)
    return s.cpu().numpy(), var.cpu().numpy()


def update_sigma_s(sigma_s, rho0, S):
    """Shared-covariance update; returns (Sigma_new, trace) (srm.py:132-142).

    ``update_sigma_s`` needs only ``var_s`` (from ``sigma_s`` and ``rho0``)
    and ``S``; the device tail computes it from a zero reduction whose S
    output is discarded.
    """
    torch = _torch()
    lib = _lib.load()
    s_dev = _dev(_as_matrix(S, "S"), torch.float64)
    k, t = s_dev.shape
    _, var, _, _ = _tail(torch.zeros((k, t), dtype=torch.float64, device="cuda"), sigma_s, rho0)
    st = s_dev.t().contiguous()
    ss = _gemm_tn(st, st)  # S S^T via the V-contraction
    new = torch.empty((k, k), dtype=torch.float64, device="cuda")
    trace = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.check(lib.srm_sigma_update(_ptr(var), k, _ptr(ss), k, k, t, _ptr(new), k, _ptr(trace), _stream()),
               "sigma_update")
    return new.cpu().numpy(), float(trace.item())


def m_step_subject(Xhat_i, S, trace_sigma_s_new):
    """Per-subject mapping and noise update (srm.py:145-155)."""
    torch = _torch()
    lib = _lib.load()
    x = _dev(_as_matrix(Xhat_i, "Xhat"), torch.float64)
    s = _dev(_as_matrix(S, "S"), torch.float64)
    a = _gemm_nt(x, s, 0.5)
    _finite(a, "A")  # kernels.py:201 via _as_matrix: non-finite A is InvalidInputError
    w = _polar(a, s.shape[0])
    n_trs = s.shape[1]
    n_voxels = x.shape[0]
    wtx = _gemm_tn(w, x)
    scal = torch.empty(2, dtype=torch.float64, device="cuda")
    ws = torch.empty(1024, dtype=torch.float64, device="cuda")
    st = _status_tensor()
    # cross = <W^T Xhat, S> (srm.py:151) and trace_ata(Xhat) (srm.py:152, with
    # the kernels.py:45 finite check) on the device, fixed summation order
    _lib.check(lib.srm_dot(_ptr(wtx), n_trs, _ptr(s), _ld(s), s.shape[0], n_trs, _ptr(scal), _ptr(ws), 8192,
                           _stream()), "dot")
    _lib.check(lib.srm_trace_ata(_ptr(x), _ld(x), n_voxels, x.shape[1], ctypes.c_void_p(scal.data_ptr() + 8),
                                 _ptr(st), _ptr(ws), 8192, _stream()), "trace_ata")
    _raise_status(st)
    cross, sq = (float(v) for v in scal.cpu().numpy())
    rho2 = (sq + n_trs * trace_sigma_s_new - 2.0 * cross) / (n_trs * n_voxels)
    return w.cpu().numpy(), max(rho2, RHO_FLOOR)


# ---------------------------------------------------------------------------
# the fit (srm.py:216-327)
# ---------------------------------------------------------------------------

def _storage_for(subjects, storage):
    if storage in ("f64", "f32"):
        return storage
    if storage not in (None, "auto"):
        raise ConfigError("storage must be 'auto', 'f64' or 'f32'")
    try:
        import torch

        tensor_t = torch.Tensor
    except ImportError:  # pragma: no cover
        tensor_t = ()
    f32 = []
    for s in subjects:
        x = s.X
        if isinstance(x, tensor_t):
            f32.append(str(x.dtype) == "torch.float32")
        elif hasattr(x, "dtype"):  # numpy arrays and pending SFAB reads (data_io.PendingMatrix)
            f32.append(np.dtype(x.dtype) == np.float32)
        else:
            f32.append(np.asarray(x).dtype == np.float32)
    return "f32" if all(f32) else "f64"


# B200 rates used by the cost model (measured on this pool: DMMA 37.1 TF/s peak, ~30 sustained
# in the contraction kernels; HBM copy 6.55 TB/s; 3xTF32 tcgen05 ~0.9 PF/s of tf32 MMA; the
# tcgen05 fp32 streaming passes sustain ~3.0 TB/s of X-hat per iteration, reductions included:
# cfg 3 17.4 ms per iteration for 2 x 25.8 GB)
_DMMA_FLOPS = 30e12
_HBM_BYTES = 6.0e12
_TF32_FLOPS = 0.9e15
_TC_STREAM_BYTES = 3.0e12
_I8_OPS = 3.2e15       # int8 tcgen05 (dense 4.5e15 nominal), as sustained by the sliced Gram
_I8_PRODUCTS = {"f64": 28, "f32": 16}  # slice pairs of the int8-sliced Gram: 7 or 4 slices per value


def gram_int8_bytes(n_voxels, n_trs, storage="f64"):
    """Device bytes of the int8 slices of the Gram path: TR-major records per
    TR and 32 voxels (256 B for fp64's seven slices, 128 B for fp32's four)
    for X^T X and the row slices of every G_i."""
    ldx = -(-n_trs // 32) * 32
    lq = -(-max(n_voxels) // 32) * (256 if storage == "f64" else 128)
    return len(n_voxels) * ldx * (lq + 12) + len(n_voxels) * ldx * ldx * 8


def choose_algorithm(n_voxels, n_trs, k, iterations, free_bytes=None, storage="f64", gram_int8=False):
    """'gram' or 'stream' from an estimate of each path's device time.

    stream: per iteration two passes over X-hat (A = X S^T / 2, B = A^T X):
            4 V T K flops per subject on the FP64 tensor pipe, or -- for fp32
            X-hat on the tcgen05 3xTF32 path -- max(HBM time of 2 reads, MMA time).
    gram:   one-time X^T X (upper 128-tiles, V T^2 flops on DMMA, or 28 / 16
            int8 slice products for fp64 / fp32 plus the slicing passes with
            ``gram_int8``), then 2 K T^2 per subject-iteration for B = S G / 2
            (a read of G's slices on the int8 path), plus one final W pass.
    """
    kp = -(-k // 8) * 8
    ldx = -(-n_trs // 32) * 32
    nt = -(-ldx // 128)
    b = 8 if storage == "f64" else 4
    tc = storage == "f32" and -(-k // 16) * 16 <= 128
    stream = 0.0
    gram = 0.0
    for v in n_voxels:
        if tc:
            np16 = -(-k // 16) * 16
            per_pass = max(v * ldx * b / _TC_STREAM_BYTES, 3 * 2.0 * v * ldx * max(np16, 128) / _TF32_FLOPS)
            stream += iterations * 2 * per_pass
            final_a = per_pass
        else:
            stream += iterations * 2 * (2.0 * v * ldx * kp) / _DMMA_FLOPS
            final_a = 2.0 * v * ldx * kp / _DMMA_FLOPS
        tiles = nt * (nt + 1) / 2 * 128 * 128 * 2.0 * v
        per_iter = 2.0 * kp * ldx * ldx / _DMMA_FLOPS
        if gram_int8:
            products = _I8_PRODUCTS[storage]
            slice_bytes = v * ldx * (8 if storage == "f64" else 4)
            one_time = products * tiles / _I8_OPS + (2.0 * v * ldx * b + slice_bytes) / _HBM_BYTES
            if kp <= 128:  # B = S G / 2 and the final W on int8 slices too
                per_iter = 8.0 * ldx * ldx / _HBM_BYTES
                final_a = max(slice_bytes / _HBM_BYTES, products * 2.0 * v * ldx * 64 / _I8_OPS)
        else:
            one_time = tiles / _DMMA_FLOPS
        gram += one_time + iterations * per_iter + final_a
    need = len(n_voxels) * ldx * ldx * 8
    if free_bytes is not None and need > 0.25 * free_bytes:
        return "stream"
    return "gram" if gram < 0.8 * stream else "stream"


def fit(subjects, config, comm=None, *, storage="auto", ordered=None, graphs=True,
        keep_on_device=False, device=None, engine_out=None, timings=None, algorithm="auto",
        tensor_cores=True, gram_int8=True, init_overlap=True, exact_polar=False, on_iteration=None):
    """Run the distributed EM; ``subjects`` are this worker's share (srm.py:216).

    Every worker calls this with the same config and its own communicator
    (``SerialCommunicator``, ``TorchCommunicator`` or any object with the
    reference protocol).  Subject data may be numpy arrays or torch tensors
    (CPU -- pinned for asynchronous upload -- or already on the GPU).

    ``storage`` picks the HBM dtype of X-hat: ``"auto"`` keeps fp32 inputs
    fp32 (half the bytes; arithmetic stays fp64), else fp64.
    ``ordered`` (default ``True``) sums subject terms in ascending global order
    on every rank -- bit-identical results for any shard layout (srm.py:193-213):
    on N > 1 ranks by TR column blocks (each rank sums every subject's block
    of T / N columns, then the K x T / N results are all-gathered) when the
    communicator has an all-to-all, else from the gathered term table.
    ``ordered=False`` all-reduces per-rank partial sums instead (opt-in: the
    rounding then depends on the sharding).
    ``timings`` (a dict) receives per-phase wall seconds (synchronising).
    ``algorithm``: ``"stream"`` (two passes over X-hat per iteration),
    ``"gram"`` (one-time X^T X, then T x T algebra per iteration) or
    ``"auto"`` (:func:`choose_algorithm`).  Both compute the reference's
    iteration exactly; they differ only in rounding.
    ``tensor_cores``: for fp32 X-hat on the streaming path, run the two passes
    as 3xTF32 tcgen05 MMAs (error ~1e-6, inside the 1e-4 fp32 tolerance);
    ``False`` keeps every contraction in fp64 on DMMA.
    ``gram_int8``: on the Gram path with fp64 X-hat, form the one-time X^T X
    from seven exact int8 slices per value on the int8 tensor cores (products
    represented to ~2^-48 of the column maxima; ~1e-14 relative to G) when
    the slices fit in device memory; ``False`` keeps it on fp64 DMMA.
    ``init_overlap`` (default): run the initial mapping (srm.py:101-118 after
    the draw) batch by batch while later subjects are still uploading;
    ``False`` runs it once after the upload (bit-identical results; ~5 ms
    more end to end on cfg 2).
    ``exact_polar``: form every polar transform from A_i itself (Householder
    TSQR + one-sided Jacobi SVD, the fp64 streaming path).  By default the
    fast routes form it from A_i^T A_i, which cannot resolve
    sigma_min / sigma_max much below 1e-3 at the fp64 tolerance; a subject
    that ill-conditioned raises a device warning and the whole fit is redone
    with ``exact_polar=True`` (on every rank), which matches the reference's
    SVD (kernels.py:190-212) and raises ``RankError`` exactly where it does.
    ``on_iteration``: called after every EM iteration with an
    :class:`IterationState` (S, Sigma_s, this worker's rho_i^2 and W_i as they
    stand after that iteration's M-step, and its log-likelihood) -- the
    per-iteration trace of the reference's loop (srm.py:254-287), for
    checking a long fit against an oracle without refitting.  Forming W_i
    reads the EM state only, so the fit is bit-identical with or without it
    (tested); it synchronises once per iteration.  A fit redone on the exact
    polar route reports its iterations again from 0.
    """
    config.validate()
    if not subjects:
        raise ConfigError("each worker needs at least one subject")
    comm = comm if comm is not None else SerialCommunicator()
    n_trs = int(subjects[0].X.shape[1])
    for s in subjects:
        if int(s.X.shape[1]) != n_trs:
            raise ShapeError(f"subject {s.subject_id} has {s.X.shape[1]} TRs, expected {n_trs}")
    if n_trs < 2:
        raise ShapeError("need at least 2 TRs")
    k = config.k
    for s in subjects:
        if int(s.X.shape[0]) < k:
            raise ShapeError(f"subject has {s.X.shape[0]} voxels, fewer than k={k} factors")
    opts = dict(storage=storage, ordered=ordered, graphs=graphs, keep_on_device=keep_on_device, device=device,
                engine_out=engine_out, timings=timings, algorithm=algorithm, tensor_cores=tensor_cores,
                gram_int8=gram_int8, init_overlap=init_overlap, on_iteration=on_iteration)
    model = _fit_pass(subjects, config, comm, exact=bool(exact_polar), **opts)
    if model is None:  # a Gram-route polar transform was out of its range on some rank
        model = _fit_pass(subjects, config, comm, exact=True, **opts)
    return model


@dataclass
class IterationState:
    """One EM iteration of a fit as seen by this worker (``fit(on_iteration=)``)."""

    iteration: int
    S: np.ndarray
    sigma_s: np.ndarray
    rho2: list
    W: list
    log_likelihood: float


def _snapshot(eng, it):
    eng.finalize()  # W_i = A_i M_i of this M-step; writes only W (and finalize scratch)
    w = hostio.to_host(eng.wout)
    return IterationState(
        iteration=it, S=eng.S.cpu().numpy(), sigma_s=eng.sigma.cpu().numpy(),
        rho2=[float(r) for r in eng.local_rho2().cpu().numpy()],
        W=[w[eng.subject_rows(j)] for j in range(eng.n_local)],
        log_likelihood=float(eng.hist[it % eng.iterations][_lib.H_LL].item()))


def _fit_pass(subjects, config, comm, *, exact, storage, ordered, graphs, keep_on_device, device, engine_out,
              timings, algorithm, tensor_cores, gram_int8, init_overlap, on_iteration):
    """One fit; None when it must be redone on the exact polar route."""
    clock = _PhaseClock(timings)
    n_trs = int(subjects[0].X.shape[1])
    k = config.k
    counts = rank_counts(comm, len(subjects))
    offset = int(sum(counts[: comm.rank]))
    n_subjects = int(sum(counts))
    if ordered is None:
        ordered = True
    # ordered multi-rank exchange: by column blocks (all-to-all of the K x T
    # terms in N blocks, ordered block sums, all-gather of K x T / N) where the
    # communicator has an all-to-all, else the gathered table;
    # SRM_B200_EXCHANGE=gather forces the gathered table
    colblock = (bool(ordered) and comm.size > 1 and hasattr(comm, "all_to_all_into")
                and os.environ.get("SRM_B200_EXCHANGE") != "gather")

    n_vox = [int(s.X.shape[0]) for s in subjects]
    store = _storage_for(subjects, storage)
    use_i8 = bool(gram_int8) and not exact
    free = None
    if use_i8 or algorithm == "auto":
        torch = _torch()
        free = _free_device_bytes(torch, device)
        x_bytes = sum(n_vox) * (-(-n_trs // 32) * 32) * (8 if store == "f64" else 4)
        use_i8 = use_i8 and gram_int8_bytes(n_vox, n_trs, store) + x_bytes < 0.6 * free
    if exact:
        algorithm = "stream"
    elif algorithm == "auto":
        algorithm = choose_algorithm(n_vox, n_trs, k, config.iterations, free,
                                     storage=store if tensor_cores else "f64", gram_int8=use_i8)
    if algorithm not in ("stream", "gram"):
        raise ConfigError("algorithm must be 'auto', 'stream' or 'gram'")
    eng = SrmEngine(n_vox, n_trs, k, config.iterations,
                    storage=store, world_size=comm.size, rank=comm.rank,
                    counts=counts, ordered=ordered, colblock=colblock, tolerance=config.tolerance is not None,
                    gram=algorithm == "gram", tc=bool(tensor_cores) and store == "f32" and not exact,
                    gram_i8=algorithm == "gram" and use_i8, exact_polar=exact, device=device)
    if engine_out is not None:
        engine_out.append(eng)
    # the init draws depend only on (seed, global index, V, k): overlap them with the upload
    pool = _draw_pool()
    ring = hostio.PinnedRing.acquire(eng.device, max(n_vox) * k * 8, nslots=min(16, len(subjects)),
                                     n_items=len(subjects))

    def draw(j):  # the srm.py:111 PCG64 stream, written straight into a pinned slot
        if not ring.wait_free(j):
            return None  # the fit was abandoned
        gen = np.random.default_rng((config.seed & 0xFFFFFFFFFFFFFFFF, offset + j))
        gen.standard_normal(out=ring.view(j, (n_vox[j], k)))
        return (ring, j)

    draws = [pool.submit(draw, j) for j in range(len(subjects))]
    futures = list(draws)  # eng.load consumes `draws`
    clock.tick("setup")
    # pipelined: upload + demean (+ X^T X) (+ the initial mapping) per batch of subjects
    # N > 1 over NCCL: the first iteration runs eagerly (it also sets up the
    # collective's channels), then {all-gather, E-step, M-step} is one graph
    # per rank.  SRM_B200_FORCE_XGRAPH=1 takes that path on one rank too (an
    # in-place one-rank all-gather), which is how it is tested on one GPU.
    force_x = comm.size == 1 and os.environ.get("SRM_B200_FORCE_XGRAPH") == "1"
    use_xgraph = graphs and (comm.size > 1 or force_x) and eng.exchange_capturable(comm)
    use_graph = graphs and comm.size == 1 and not use_xgraph
    try:
        eng.load([s.X for s in subjects], gaussians=draws, gram=True, init=init_overlap, capture=use_graph)
    except BaseException:
        # wake and drain the draw workers before the ring is reused by another fit
        ring.cancel()
        for f in futures:
            f.cancel()
        for f in futures:
            if not f.cancelled():
                try:
                    f.result()
                except Exception:  # noqa: BLE001
                    pass
        ring.release()
        eng.close()
        raise
    ring.release()
    clock.tick("load")
    if init_overlap:
        eng.set_iteration(0)
    else:
        eng.init_kernels()
    if not keep_on_device:
        eng.start_mu_readback()  # mu is final after the demean: read it back under the EM
    clock.tick("init")

    n_done = 0
    for it in range(config.iterations):
        if use_graph:
            eng.replay()  # one EM iteration; the graph was captured during the upload
        elif use_xgraph and it >= 1:
            if it == 1:
                eng.capture_exchange(comm, force=force_x)
            eng.replay_exchange()
        elif use_xgraph:
            eng.exchange(comm, force=force_x)
            eng.step(None)
        else:
            eng.step(comm)
        n_done = it + 1
        if config.tolerance is not None or on_iteration is not None:
            # one copy + one stream synchronisation per iteration: status and |dS|, |S_prev|;
            # a polar-conditioning warning first (the pass is redone), then errors
            code, arg, warn, sdiff, sprev = eng.poll(it)
            if not exact and any_rank(comm, warn != 0):
                eng.close()
                return None
            if code:
                raise from_status(code, arg=arg)
            if on_iteration is not None:
                state = _snapshot(eng, it)
                if not exact and any_rank(comm, eng.status()[3] != 0):  # the snapshot's final transform
                    eng.close()
                    return None
                on_iteration(state)
            if config.tolerance is not None and it >= 1 and sdiff / max(sprev, 1e-300) < config.tolerance:
                break
    clock.tick("em")
    if keep_on_device:
        eng.finalize()
        wout = None
    else:
        # W_i of earlier subjects read back while later ones are formed
        wout = eng.finalize_to_host()
    code, arg, _, warn = eng.status()  # warnings are sticky: this covers init, every M-step and the final W
    if not exact and any_rank(comm, warn != 0):
        eng.close()
        return None
    if code:
        raise from_status(code, arg=arg)
    clock.tick("finalize")
    model = _collect(eng, subjects, comm, offset, n_subjects, n_done, keep_on_device, wout)
    clock.tick("collect")
    return model


_FREE_BASE = {}


def _free_device_bytes(torch, device):
    """Device bytes a fit can still allocate: cudaMemGetInfo once per device
    (it costs milliseconds), plus what torch's caching allocator had reserved
    then, minus what torch has allocated now (reserved-but-free blocks are
    reusable, so they count as free)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if idx not in _FREE_BASE:
        free, _ = torch.cuda.mem_get_info(idx)
        _FREE_BASE[idx] = free + torch.cuda.memory_reserved(idx)
    return max(0, _FREE_BASE[idx] - torch.cuda.memory_allocated(idx))


_DRAW_POOL = None


def _draw_pool():
    """Host threads for the init draws, kept across fits (thread start-up is
    ~0.1 ms per thread on the fit's critical path otherwise)."""
    global _DRAW_POOL
    if _DRAW_POOL is None:
        _DRAW_POOL = ThreadPoolExecutor(max(1, os.cpu_count() or 1), thread_name_prefix="srm-draw")
    return _DRAW_POOL


class _PhaseClock:
    def __init__(self, out):
        self.out = out
        self.t = time.perf_counter()

    def tick(self, name):
        if self.out is None:
            return
        _torch().cuda.synchronize()
        now = time.perf_counter()
        self.out[name] = self.out.get(name, 0.0) + now - self.t
        self.t = now


def _collect(eng, subjects, comm, offset, n_subjects, n_done, keep_on_device, wout=None):
    torch = _torch()
    if not keep_on_device:
        rho2_np, hist, S_np, sigma_np = eng.small_results_to_host(n_done)
        rho2_local = torch.from_numpy(rho2_np.copy())
    else:
        rho2_local = eng.local_rho2().clone()
    # final rho^2 gather + rho0 refresh (srm.py:289-313)
    if comm.size > 1:
        m = max(eng.counts)
        mine = torch.zeros(m, dtype=torch.float64, device=eng.device)
        mine[: eng.n_local] = rho2_local
        if hasattr(comm, "all_gather_into"):
            allr = torch.empty(comm.size * m, dtype=torch.float64, device=eng.device)
            comm.all_gather_into(allr, mine)
            parts = [allr[r * m: r * m + eng.counts[r]] for r in range(comm.size)]
            rho2_all = torch.cat(parts).cpu().numpy()
        else:
            blobs = comm.gather(rho2_local.cpu().numpy().tobytes())
            tab = None
            if comm.rank == 0:
                tab = np.concatenate([np.frombuffer(b, np.float64) for b in blobs])[None, :]
            rho2_all = comm.broadcast(tab)[0]
    else:
        rho2_all = rho2_local.cpu().numpy()
    rho0 = float(np.add.reduce(1.0 / rho2_all))
    if keep_on_device:
        hist = eng.hist[:n_done].cpu().numpy()
    rho2_hist = hist[:, _lib.H_RHO2: _lib.H_RHO2 + eng.n_local]
    objective = [float(np.mean(r)) for r in rho2_hist]
    lls = [float(x) for x in hist[:, _lib.H_LL]]
    if keep_on_device:
        W = [eng.wout[eng.subject_rows(j)] for j in range(eng.n_local)]
        mu = [eng.mu[eng.subject_rows(j)] for j in range(eng.n_local)]
        S = eng.S.clone()
        sigma = eng.sigma.clone()
    else:
        # W lands by DMA in pinned memory from torch's caching host allocator
        # (reused once an earlier model is released); the arrays are views of it
        if wout is None:
            wout = hostio.to_pinned(eng.wout)
        muh = eng.mu_host()  # pinned too; mu_i are views of it like W_i
        W = [wout[eng.subject_rows(j)] for j in range(eng.n_local)]
        mu = [muh[eng.subject_rows(j)] for j in range(eng.n_local)]
        S = np.array(S_np)
        sigma = np.array(sigma_np)
    model = SrmModel(
        subject_ids=[s.subject_id for s in subjects],
        subject_indices=list(range(offset, offset + len(subjects))),
        W=W,
        rho2=[float(r) for r in rho2_local.cpu().numpy()],
        mu=mu,
        S=S,
        rho0=rho0,
        n_subjects=n_subjects,
        sigma_s=sigma if comm.rank == 0 else None,
        rho2_all=np.asarray(rho2_all) if comm.rank == 0 else None,
        objective_trace=objective,
        log_likelihood=lls,
        device_state=eng if keep_on_device else None,
    )
    if not keep_on_device:
        eng.close()
    return model


# ---------------------------------------------------------------------------
# transforms (srm.py:330-338)
# ---------------------------------------------------------------------------

def _model_arrays(model, i):
    """(W_i, mu_i) of a fitted model on the device; IndexError like list indexing."""
    torch = _torch()
    if not -len(model.W) <= i < len(model.W):
        raise IndexError(f"subject index {i} out of range for {len(model.W)} held subjects")
    w = _dev(model.W[i], torch.float64)
    mu = _dev(model.mu[i], torch.float64).reshape(-1)
    return w, mu


def _project_dev(model, i, X):
    torch = _torch()
    lib = _lib.load()
    w, mu = _model_arrays(model, i)
    x = X if isinstance(X, torch.Tensor) else np.asarray(X)
    if x.ndim == 1:
        x = x.reshape(-1, 1)
    v, k = w.shape
    if x.shape[0] != v:
        raise ShapeError(f"subject {i} has {v} voxels, got volumes of {x.shape[0]}")
    xd = _dev(x)
    t = xd.shape[1]
    out = torch.empty((k, t), dtype=torch.float64, device=w.device)
    ws, nb = _workspace(v, k, t)
    dt = _lib.SRM_F64 if xd.dtype == torch.float64 else _lib.SRM_F32
    _lib.check(lib.srm_project(_ptr(w), _ld(w), _ptr(xd), dt, _ld(xd), _ptr(mu), v, k, t, _ptr(out), t,
                               _ptr(ws), nb, _stream()), "project")
    return out


def project_batch(model, i, X):
    """Map V_i x T' volumes of held subject ``i`` into the shared space:
    W_i^T (X - mu_i) (srm.py:330-333 over a block of columns; K x T')."""
    return _project_dev(model, i, X).cpu().numpy()


def map_between_batch(model, i, j, X):
    """Map V_i x T' volumes of subject ``i`` into subject ``j``'s voxel space:
    W_j W_i^T (X - mu_i) + mu_j (srm.py:336-338 over a block; V_j x T')."""
    torch = _torch()
    lib = _lib.load()
    z = _project_dev(model, i, X)
    wj, muj = _model_arrays(model, j)
    vj, k = wj.shape
    t = z.shape[1]
    out = torch.empty((vj, t), dtype=torch.float64, device=wj.device)
    _lib.check(lib.srm_unproject(_ptr(wj), _ld(wj), _ptr(z), _ld(z), _ptr(muj), vj, k, t, _ptr(out), t,
                                 _stream()), "map_between")
    return out.cpu().numpy()


def project(model, i, x):
    """Map one volume of held subject ``i`` into the shared space (srm.py:330-333)."""
    torch = _torch()
    xv = x.reshape(-1) if isinstance(x, torch.Tensor) else np.asarray(x, dtype=np.float64).ravel()
    return project_batch(model, i, xv.reshape(-1, 1)).reshape(-1)


def map_between(model, i, j, x):
    """Map a volume of subject ``i`` into subject ``j``'s voxel space (srm.py:336-338)."""
    torch = _torch()
    xv = x.reshape(-1) if isinstance(x, torch.Tensor) else np.asarray(x, dtype=np.float64).ravel()
    return map_between_batch(model, i, j, xv.reshape(-1, 1)).reshape(-1)
