"""CPU oracle for the SRM EM hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy/scipy restatement of the reference
``factorfit.srm`` fit (``/root/reference/pkg/src/factorfit/srm.py``) and
the dense helpers it calls (``kernels.py``).  It exists so that

* ``tests/`` can check the CUDA path against the reference algorithm on
  identical inputs and initialisation,
* ``bench.py`` can time the reference's own CPU arithmetic
  (``--impl reference`` and the ``cpu_baseline`` leg), and
* ``__graft_entry__.smoke()`` can check one tiny CUDA fit.

Nothing in ``paper_1608_04647_b200/`` imports this file; the product
path fails loudly when its CUDA library is missing instead of falling
back here.

Parity pin: every function below is checked against golden vectors that
``tests/golden/make_golden.py`` produced by importing the real reference
package (``tests/test_oracle_golden.py``).  The per-iteration EM driver
``run_em`` reproduces ``factorfit.srm.fit`` on a serial communicator
bit-for-bit (same numpy/LAPACK calls in the same order).

The step functions intentionally keep the reference's cost structure
(four passes over X-hat per iteration, the loop-invariant ``trace_ata``
recompute and the V x K SVD), so timing them times the reference.
"""

import math

import numpy as np
from scipy.linalg import lapack

RHO_FLOOR = 1e-12          # srm.py:48
RANK_TOLERANCE = 1e-12     # kernels.py:32
MAX_NAIVE_VOXELS = 2000    # reference.py:23


class OracleError(Exception):
    """Raised where the reference raises one of its FactorFitError types.

    ``kind`` names the reference exception class (``"RankError"``,
    ``"DefinitenessError"``, ``"InvalidInputError"``, ``"ShapeError"``),
    ``pivot`` mirrors ``DefinitenessError.pivot``.
    """

    def __init__(self, kind, message, pivot=None):
        super().__init__(f"{kind}: {message}")
        self.kind = kind
        self.pivot = pivot


# --------------------------------------------------------------------------
# dense helpers (kernels.py)
# --------------------------------------------------------------------------

def _f64(a, name="matrix"):
    """kernels.py:39-47 -- contiguous float64 2-D view, finite entries."""
    out = np.ascontiguousarray(a, dtype=np.float64)
    if out.ndim != 2 or out.shape[0] < 1 or out.shape[1] < 1:
        raise OracleError("ShapeError", f"{name} must be a non-empty 2-D array")
    if not np.all(np.isfinite(out)):
        raise OracleError("InvalidInputError", f"{name} contains non-finite entries")
    return out


def sum_of_squares(a):
    """kernels.py:152-155 ``trace_ata``."""
    a = _f64(a, "A")
    return float(np.einsum("ij,ij->", a, a))


def shift_diagonal(a, c):
    """kernels.py:158-165 ``add_diag``."""
    out = _f64(a, "A").copy()
    out[np.diag_indices_from(out)] += c
    return out


def chol_inverse(a):
    """kernels.py:168-187 ``spd_inverse``: dpotrf + dpotri, symmetrised."""
    a = _f64(a, "A")
    if a.shape[0] != a.shape[1]:
        raise OracleError("ShapeError", "spd inverse needs a square matrix")
    factor, info = lapack.dpotrf(a, lower=1, overwrite_a=0)
    if info > 0:
        raise OracleError("DefinitenessError", "not positive definite", pivot=info - 1)
    inv, info = lapack.dpotri(factor, lower=1)
    if info != 0:
        raise OracleError("DefinitenessError", "inverse failed", pivot=abs(info) - 1)
    low = np.tril(inv)
    full = low + np.tril(inv, -1).T
    return 0.5 * (full + full.T)


def orthogonal_polar(a):
    """kernels.py:190-212 ``polar_orthogonal``: gesdd, rank check, sign fix."""
    a = _f64(a, "A")
    n_rows, n_cols = a.shape
    if n_rows < n_cols:
        raise OracleError("ShapeError", "polar factor needs rows >= cols")
    u, sv, vt = np.linalg.svd(a, full_matrices=False)
    if sv[0] == 0.0 or sv[-1] < RANK_TOLERANCE * sv[0]:
        raise OracleError("RankError", "rank-deficient input")
    for j in range(n_cols):
        if vt[j, np.argmax(np.abs(vt[j]))] < 0.0:
            vt[j] = -vt[j]
            u[:, j] = -u[:, j]
    return u @ vt


# --------------------------------------------------------------------------
# SRM steps (srm.py)
# --------------------------------------------------------------------------

def center_rows(x):
    """srm.py:94-98 ``demean``: (X - row mean, row mean), upcast to fp64."""
    x = np.asarray(x, dtype=np.float64)
    mu = x.mean(axis=1)
    return x - mu[:, None], mu


def initial_mapping(n_voxels, k, seed, subject_index):
    """srm.py:101-113 ``init_subject``: polar(N(0,1)) from PCG64((seed, idx))."""
    if n_voxels < k:
        raise OracleError("ShapeError", "fewer voxels than factors")
    gen = np.random.default_rng((seed & 0xFFFFFFFFFFFFFFFF, subject_index))
    return orthogonal_polar(gen.standard_normal((n_voxels, k))), 1.0


def initial_gaussian(n_voxels, k, seed, subject_index):
    """The N(0,1) draw inside ``init_subject`` before its polar factor."""
    gen = np.random.default_rng((seed & 0xFFFFFFFFFFFFFFFF, subject_index))
    return gen.standard_normal((n_voxels, k))


def local_term(w, rho2, xhat):
    """srm.py:116-118 ``e_step_local``: W^T Xhat / rho^2."""
    return (w.T @ xhat) / rho2


def shared_posterior(reduced, sigma_s, rho0):
    """srm.py:121-129 ``e_step_global`` -> (S, var_s)."""
    k = sigma_s.shape[0]
    var_s = chol_inverse(shift_diagonal(chol_inverse(sigma_s), rho0))
    s = (sigma_s.T @ (np.eye(k) - rho0 * var_s)) @ reduced
    return s, var_s


def shared_covariance(sigma_s, rho0, s):
    """srm.py:132-142 ``update_sigma_s`` -> (Sigma_new, trace)."""
    var_s = chol_inverse(shift_diagonal(chol_inverse(sigma_s), rho0))
    new = var_s + (s @ s.T) / s.shape[1]
    new = 0.5 * (new + new.T)
    return new, float(np.trace(new))


def subject_update(xhat, s, trace_new):
    """srm.py:145-155 ``m_step_subject`` -> (W_new, rho2_new)."""
    a = 0.5 * (xhat @ s.T)
    w = orthogonal_polar(a)
    n_trs = s.shape[1]
    n_vox = xhat.shape[0]
    cross = float(np.einsum("kt,kt->", w.T @ xhat, s))
    rho2 = (sum_of_squares(xhat) + n_trs * trace_new - 2.0 * cross) / (n_trs * n_vox)
    return w, max(rho2, RHO_FLOOR)


def ordered_reduce(terms, rho2s):
    """srm.py:193-213 ``_accumulate``: ascending subject order."""
    reduced = terms[0].copy()
    rho0 = 1.0 / rho2s[0]
    for term, r in zip(terms[1:], rho2s[1:]):
        reduced += term
        rho0 += 1.0 / r
    return reduced, rho0


# --------------------------------------------------------------------------
# log-likelihood
# --------------------------------------------------------------------------

def naive_loglik(ws, rho2s, sigma_s, xhats):
    """reference.py:55-65 ``naive_log_likelihood`` (explicit V x V Phi)."""
    v_total = sum(w.shape[0] for w in ws)
    if v_total > MAX_NAIVE_VOXELS:
        raise OracleError("InvalidInputError", "naive oracle refuses large V")
    w = np.vstack(ws)
    psi = np.concatenate([np.full(wi.shape[0], r) for wi, r in zip(ws, rho2s)])
    xhat = np.vstack(xhats)
    n_trs = xhat.shape[1]
    phi = w @ sigma_s @ w.T
    phi[np.diag_indices_from(phi)] += psi
    chol = np.linalg.cholesky(phi)
    logdet = 2.0 * float(np.sum(np.log(np.diag(chol))))
    solved = np.linalg.solve(chol, xhat)
    quad = float(np.einsum("ij,ij->", solved, solved))
    return -0.5 * (n_trs * (v_total * np.log(2.0 * np.pi) + logdet) + quad)


def naive_posterior(ws, rho2s, sigma_s, xhats):
    """reference.py:43-52 ``naive_posterior`` (explicit V x V inverse)."""
    w = np.vstack(ws)
    psi = np.concatenate([np.full(wi.shape[0], r) for wi, r in zip(ws, rho2s)])
    xhat = np.vstack(xhats)
    phi = w @ sigma_s @ w.T
    phi[np.diag_indices_from(phi)] += psi
    phi_inv = chol_inverse(phi)
    proj = sigma_s.T @ w.T @ phi_inv
    s = proj @ xhat
    var_s = sigma_s - proj @ w @ sigma_s
    return s, 0.5 * (var_s + var_s.T)


def woodbury_loglik(reduced, rho0, sigma_s, rho2s, n_voxels, sqnorms, n_trs):
    """Marginal log-likelihood through the determinant lemma.

    With Z = sum_i W_i^T Xhat_i / rho_i^2 (``reduced``) and
    P = Sigma_s^{-1} + rho0 I:
        LL = -1/2 [ T (sum V log 2pi + sum_i V_i log rho_i^2 + log|Sigma_s|
                       + log|P|) + sum_i |Xhat_i|^2 / rho_i^2 - tr(Z^T P^{-1} Z) ]
    Equals ``naive_loglik`` whenever every W_i is orthonormal.
    """
    v_total = float(sum(n_voxels))
    l_sigma = np.linalg.cholesky(sigma_s)
    logdet_sigma = 2.0 * float(np.sum(np.log(np.diag(l_sigma))))
    prec = shift_diagonal(chol_inverse(sigma_s), rho0)
    l_prec = np.linalg.cholesky(prec)
    logdet_prec = 2.0 * float(np.sum(np.log(np.diag(l_prec))))
    var_s = chol_inverse(prec)
    logdet_psi = float(sum(v * math.log(r) for v, r in zip(n_voxels, rho2s)))
    quad = float(sum(q / r for q, r in zip(sqnorms, rho2s)))
    quad -= float(np.einsum("kt,kt->", reduced, var_s @ reduced))
    return -0.5 * (n_trs * (v_total * math.log(2.0 * math.pi) + logdet_psi
                            + logdet_sigma + logdet_prec) + quad)


# --------------------------------------------------------------------------
# the EM driver (srm.py:216-327, serial communicator)
# --------------------------------------------------------------------------

def run_em(xs, k, iterations, seed=0, tolerance=None, record=True,
           init_ws=None):
    """Serial restatement of ``srm.fit`` with per-iteration records.

    Returns a dict with the final model fields (``W``, ``rho2``, ``mu``,
    ``S``, ``sigma_s``, ``rho0``, ``objective``) and, when ``record`` is
    true, ``iters``: one dict per EM iteration holding the S, Sigma_s,
    trace, rho2 vector, W list and the Woodbury log-likelihood of the
    parameters that entered that iteration's E-step.
    """
    n_trs = xs[0].shape[1]
    centered = [center_rows(x) for x in xs]
    xhats = [c[0] for c in centered]
    mus = [c[1] for c in centered]
    if init_ws is None:
        init_ws = [initial_mapping(xh.shape[0], k, seed, j)[0]
                   for j, xh in enumerate(xhats)]
    ws = [np.array(w, dtype=np.float64) for w in init_ws]
    rho2s = [1.0] * len(xhats)
    sigma_s = np.eye(k)
    s_prev = None
    s = None
    objective = []
    records = []
    n_vox = [xh.shape[0] for xh in xhats]
    sqnorms = [sum_of_squares(xh) for xh in xhats] if record else None
    for _ in range(iterations):
        terms = [local_term(ws[j], rho2s[j], xhats[j]) for j in range(len(xhats))]
        reduced, rho0 = ordered_reduce(terms, rho2s)
        ll = (woodbury_loglik(reduced, rho0, sigma_s, rho2s, n_vox, sqnorms, n_trs)
              if record else None)
        s, _ = shared_posterior(reduced, sigma_s, rho0)
        sigma_s, trace_new = shared_covariance(sigma_s, rho0, s)
        for j in range(len(xhats)):
            ws[j], rho2s[j] = subject_update(xhats[j], s, trace_new)
        objective.append(float(np.mean(rho2s)))
        if record:
            records.append({
                "S": s.copy(), "sigma_s": sigma_s.copy(), "trace": trace_new,
                "rho0": rho0, "rho2": np.array(rho2s), "W": [w.copy() for w in ws],
                "ll": ll,
            })
        if tolerance is not None:
            stop = False
            if s_prev is not None:
                denom = max(float(np.linalg.norm(s_prev)), 1e-300)
                stop = float(np.linalg.norm(s - s_prev)) / denom < tolerance
            s_prev = s.copy()
            if stop:
                break
    rho2_all = np.array(rho2s)
    return {
        "W": ws, "rho2": list(rho2s), "mu": mus, "S": s, "sigma_s": sigma_s,
        "rho0": float(np.add.reduce(1.0 / rho2_all)), "rho2_all": rho2_all,
        "objective": objective, "iters": records,
    }


def _update_keep_product(xhat, s, trace_new, sqnorm):
    """``subject_update`` keeping W_new^T Xhat (srm.py:151), which is also the
    next iteration's ``e_step_local`` product (srm.py:118): the same matmul of
    the same operands, so reusing it is bit-identical; ``sqnorm`` is the
    loop-invariant ``trace_ata(Xhat)`` (srm.py:152)."""
    a = 0.5 * (xhat @ s.T)
    w = orthogonal_polar(a)
    wtx = w.T @ xhat
    cross = float(np.einsum("kt,kt->", wtx, s))
    n_trs, n_vox = s.shape[1], xhat.shape[0]
    rho2 = (sqnorm + n_trs * trace_new - 2.0 * cross) / (n_trs * n_vox)
    return w, max(rho2, RHO_FLOOR), wtx


def em_iterations(xs, k, iterations, seed=0, workers=1, keep_xhat=True):
    """``run_em`` for BASELINE-sized configs: yields one record per EM
    iteration (S, Sigma_s, trace, rho0, rho2, W list, Woodbury LL) instead of
    keeping them all.

    Same steps and arithmetic as ``run_em`` (bit-identical records; tested),
    restructured for memory and time only:

    * the loop-invariant ``trace_ata(Xhat_i)`` is computed once, and the
      M-step's W_new^T Xhat product is reused as the next E-step term (the
      reference computes both twice, with identical results);
    * ``workers`` > 1 runs the per-subject steps in threads with one BLAS
      thread each (the ordered reduction stays in ascending subject order);
    * ``keep_xhat=False`` keeps only the caller's arrays and re-forms
      Xhat_i = demean(X_i) (srm.py:94-98, deterministic) each time it is
      read, so a config whose fp64 Xhat exceeds host RAM still fits.
    """
    from concurrent.futures import ThreadPoolExecutor

    n = len(xs)
    n_trs = xs[0].shape[1]

    def xhat(j):
        return cached[j] if keep_xhat else center_rows(xs[j])[0]

    limits = None
    if workers > 1:
        from threadpoolctl import threadpool_limits

        limits = threadpool_limits(limits=1)
    try:
        pool = ThreadPoolExecutor(max(1, workers))
        cached = list(pool.map(lambda x: center_rows(x)[0], xs)) if keep_xhat else None
        n_vox = [x.shape[0] for x in xs]

        def start(j):
            xh = xhat(j)
            w = initial_mapping(xh.shape[0], k, seed, j)[0]
            return w, w.T @ xh, sum_of_squares(xh)

        first = list(pool.map(start, range(n)))
        ws = [f[0] for f in first]
        wtx = [f[1] for f in first]
        sqnorms = [f[2] for f in first]
        del first
        rho2s = [1.0] * n
        sigma_s = np.eye(k)
        for it in range(iterations):
            terms = [wtx[j] / rho2s[j] for j in range(n)]  # local_term, srm.py:118
            reduced, rho0 = ordered_reduce(terms, rho2s)
            del terms
            ll = woodbury_loglik(reduced, rho0, sigma_s, rho2s, n_vox, sqnorms, n_trs)
            s, _ = shared_posterior(reduced, sigma_s, rho0)
            sigma_s, trace_new = shared_covariance(sigma_s, rho0, s)
            out = list(pool.map(lambda j: _update_keep_product(xhat(j), s, trace_new, sqnorms[j]), range(n)))
            ws = [o[0] for o in out]
            rho2s = [o[1] for o in out]
            wtx = [o[2] for o in out]
            del out
            yield {"it": it, "S": s, "sigma_s": sigma_s.copy(), "trace": trace_new, "rho0": rho0,
                   "rho2": np.array(rho2s), "W": ws, "ll": ll}
    finally:
        if limits is not None:
            limits.restore_original_limits()


def final_loglik(ws, rho2s, sigma_s, xhats):
    """Woodbury log-likelihood of a fitted model (post-M-step parameters)."""
    terms = [local_term(w, r, xh) for w, r, xh in zip(ws, rho2s, xhats)]
    reduced, rho0 = ordered_reduce(terms, rho2s)
    return woodbury_loglik(reduced, rho0, sigma_s, rho2s,
                           [xh.shape[0] for xh in xhats],
                           [sum_of_squares(xh) for xh in xhats], xhats[0].shape[1])


def flops_per_subject_iteration(n_voxels, n_trs, k):
    """cli.py:64-72 analytic flop model of one subject-iteration."""
    v, t, k = float(n_voxels), float(n_trs), float(k)
    return 2.0 * (2.0 * v * t * k) + 2.0 * v * k * k + (2.0 * v * k * k - (2.0 / 3.0) * k ** 3)
