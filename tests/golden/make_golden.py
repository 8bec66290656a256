"""Generate the SRM golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``factorfit`` from ``/root/reference/pkg/src`` read-only and
stores inputs plus the reference's outputs in ``tests/golden/*.npz``.
The committed fixtures pin ``oracle/srm_oracle.py`` (CPU tests) and,
through the oracle, the CUDA path (GPU tests).  Nothing at test time
reads /root/reference.
"""

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _ref():
    sys.path.insert(0, str(REF_SRC))
    from factorfit import kernels, reference, srm  # noqa: E402
    from factorfit.collectives import SerialCommunicator  # noqa: E402
    from factorfit.data_io import SubjectData  # noqa: E402
    return srm, kernels, reference, SerialCommunicator, SubjectData


def recipe_subjects(rng, n_subjects, n_voxels, n_trs, k, smooth_sigma=None,
                    dtype=np.float64):
    """BASELINE.json generative recipe at small size (numpy stream)."""
    shared = rng.standard_normal((k, n_trs))
    xs = []
    for _ in range(n_subjects):
        g = rng.standard_normal((n_voxels, k))
        if smooth_sigma:
            from scipy.ndimage import gaussian_filter1d
            g = gaussian_filter1d(g, smooth_sigma, axis=0, mode="constant")
        q, _ = np.linalg.qr(g)
        rho = rng.uniform(0.5, 1.5)
        x = q @ shared + rho * rng.standard_normal((n_voxels, n_trs))
        x = x - x.mean(axis=1, keepdims=True)
        xs.append(x.astype(dtype))
    return xs


def em_trace(srm, reference, xs, k, seed, iterations, naive=True):
    """Step-driven loop (test_acceptance.py:116-141 pattern), bit-identical to srm.fit."""
    xhats = [srm.demean(x)[0] for x in xs]
    cfg = srm.SrmConfig(k=k, seed=seed)
    ws = [srm.init_subject(xh.shape[0], cfg, i)[0] for i, xh in enumerate(xhats)]
    rho2 = [1.0] * len(xs)
    sigma_s = np.eye(k)
    out = {"W0": ws}
    per = []
    for _ in range(iterations):
        lls = (reference.naive_log_likelihood(ws, rho2, sigma_s, xhats)
               if naive else np.nan)
        terms = [srm.e_step_local(ws[i], rho2[i], xhats[i]) for i in range(len(xs))]
        reduced = terms[0].copy()
        rho0 = 1.0 / rho2[0]
        for t, r in zip(terms[1:], rho2[1:]):
            reduced += t
            rho0 += 1.0 / r
        S, var_s = srm.e_step_global(reduced, sigma_s, rho0)
        sigma_s, trace = srm.update_sigma_s(sigma_s, rho0, S)
        for i in range(len(xs)):
            ws[i], rho2[i] = srm.m_step_subject(xhats[i], S, trace)
        per.append({"S": S, "sigma_s": sigma_s, "trace": trace, "rho0": rho0,
                    "rho2": np.array(rho2), "W": [w.copy() for w in ws],
                    "ll_naive": lls, "reduced": reduced, "var_s": var_s})
    out["per"] = per
    return out


def save_trace(name, xs, k, seed, iterations, srm, reference, SerialCommunicator,
               SubjectData, naive=True):
    tr = em_trace(srm, reference, xs, k, seed, iterations, naive=naive)
    model = srm.fit([SubjectData(f"s{i}", x) for i, x in enumerate(xs)],
                    srm.SrmConfig(k=k, iterations=iterations, seed=seed),
                    SerialCommunicator())
    d = {"k": k, "seed": seed, "iterations": iterations, "n_subjects": len(xs)}
    for i, x in enumerate(xs):
        d[f"X{i}"] = x
        d[f"W0_{i}"] = tr["W0"][i]
        d[f"fit_W{i}"] = model.W[i]
        d[f"fit_mu{i}"] = model.mu[i]
    d["fit_S"] = model.S
    d["fit_sigma_s"] = model.sigma_s
    d["fit_rho2"] = np.array(model.rho2)
    d["fit_rho0"] = model.rho0
    d["fit_objective"] = np.array(model.objective_trace)
    for it, p in enumerate(tr["per"]):
        for key in ("S", "sigma_s", "trace", "rho0", "rho2", "ll_naive", "reduced", "var_s"):
            d[f"it{it}_{key}"] = p[key]
        for i, w in enumerate(p["W"]):
            d[f"it{it}_W{i}"] = w
    if naive:
        xhats = [srm.demean(x)[0] for x in xs]
        d["final_ll_naive"] = reference.naive_log_likelihood(
            model.W, model.rho2, model.sigma_s, xhats)
    np.savez_compressed(OUT / f"{name}.npz", **d)
    print(f"wrote {name}.npz")


def main():
    srm, kernels, reference, SerialCommunicator, SubjectData = _ref()

    # ---- dense kernels (kernels.py) --------------------------------------
    rng = np.random.default_rng(20240601)
    d = {}
    for j, n in enumerate((1, 3, 7, 16, 50)):
        c = rng.standard_normal((n, n))
        spd = c @ c.T + 0.5 * np.eye(n)
        d[f"spd_in{j}"] = spd
        d[f"spd_out{j}"] = kernels.spd_inverse(spd)
    # cond ~1e6 (test_kernels.py:119-126 pattern)
    q, _ = np.linalg.qr(rng.standard_normal((8, 8)))
    ill = q @ np.diag(np.logspace(0, 6, 8)) @ q.T
    d["spd_ill_in"] = ill
    d["spd_ill_out"] = kernels.spd_inverse(ill)
    # indefinite: failing pivot
    bad = np.eye(5)
    bad[3, 3] = -1.0
    try:
        kernels.spd_inverse(bad)
    except Exception as exc:  # DefinitenessError
        d["spd_bad_in"] = bad
        d["spd_bad_pivot"] = exc.pivot
    for j, (r, c) in enumerate(((5, 5), (40, 3), (300, 12), (400, 30))):
        a = rng.standard_normal((r, c))
        d[f"polar_in{j}"] = a
        d[f"polar_out{j}"] = kernels.polar_orthogonal(a)
    a = rng.standard_normal((30, 7))
    d["tata_in"] = a
    d["tata_out"] = kernels.trace_ata(a)
    # demean exact examples (test_srm.py:26-41)
    d["demean_in"] = np.array([[1.0, 3.0], [2.0, 2.0]])
    xh, mu = srm.demean(d["demean_in"])
    d["demean_xhat"], d["demean_mu"] = xh, mu
    x = rng.normal(5.0, 2.0, (100, 20))
    d["demean_in2"] = x
    d["demean_xhat2"], d["demean_mu2"] = srm.demean(x)
    # init_subject (srm.py:101-113)
    for j, (v, k, seed, idx) in enumerate(((10, 3, 42, 5), (200, 8, 0, 0), (64, 64, 7, 3),
                                           (1500, 20, 0, 39))):
        d[f"init_args{j}"] = np.array([v, k, seed, idx])
        d[f"init_W{j}"] = srm.init_subject(v, srm.SrmConfig(k=k, seed=seed), idx)[0]
    np.savez_compressed(OUT / "kernels.npz", **d)
    print("wrote kernels.npz")

    # ---- single steps vs naive oracle (test_srm.py:66-177) ---------------
    rng = np.random.default_rng(5)
    d = {}
    n_s, n_v, n_t, k = 3, 20, 15, 4
    ws = [kernels.polar_orthogonal(rng.standard_normal((n_v, k))) for _ in range(n_s)]
    rho2 = rng.uniform(0.3, 2.5, n_s)
    c = rng.standard_normal((k, k))
    sigma = c @ c.T + np.eye(k)
    xhats = [srm.demean(rng.standard_normal((n_v, n_t)))[0] for _ in range(n_s)]
    for i in range(n_s):
        d[f"W{i}"], d[f"Xhat{i}"] = ws[i], xhats[i]
        d[f"local{i}"] = srm.e_step_local(ws[i], rho2[i], xhats[i])
    d["rho2"], d["sigma_s"] = rho2, sigma
    reduced = sum(srm.e_step_local(W, r, X) for W, r, X in zip(ws, rho2, xhats))
    rho0 = sum(1.0 / r for r in rho2)
    S, var_s = srm.e_step_global(reduced, sigma, rho0)
    d["reduced"], d["rho0"], d["S"], d["var_s"] = reduced, rho0, S, var_s
    d["S_naive"], d["var_naive"] = reference.naive_posterior(ws, list(rho2), sigma, xhats)
    sig_new, trace = srm.update_sigma_s(sigma, rho0, S)
    d["sigma_new"], d["trace"] = sig_new, trace
    for i in range(n_s):
        w_new, r_new = srm.m_step_subject(xhats[i], S, trace)
        d[f"mW{i}"], d[f"mrho2_{i}"] = w_new, r_new
    d["ll_naive"] = reference.naive_log_likelihood(ws, list(rho2), sigma, xhats)
    np.savez_compressed(OUT / "steps.npz", **d)
    print("wrote steps.npz")

    # ---- whole-fit traces -------------------------------------------------
    rng = np.random.default_rng(2024)
    xs = recipe_subjects(rng, 3, 60, 24, 4)
    save_trace("em_small", xs, 4, 0, 12, srm, reference, SerialCommunicator, SubjectData)

    # unequal voxel counts, non-centred data with per-voxel means
    rng = np.random.default_rng(77)
    shared = rng.standard_normal((3, 20))
    xs = []
    for v in (45, 30, 70, 38):
        w = kernels.polar_orthogonal(rng.standard_normal((v, 3)))
        xs.append(w @ shared + rng.standard_normal(v)[:, None]
                  + 0.3 * rng.standard_normal((v, 20)))
    save_trace("em_ragged", xs, 3, 5, 10, srm, reference, SerialCommunicator, SubjectData)

    # BASELINE recipe, fp32 inputs upcast by the reference
    rng = np.random.default_rng(99)
    xs = recipe_subjects(rng, 4, 400, 64, 6, dtype=np.float32)
    save_trace("em_recipe_f32", xs, 6, 0, 6, srm, reference, SerialCommunicator,
               SubjectData, naive=False)

    # smoothed-W recipe (cfg 4 structure) at small size
    rng = np.random.default_rng(4)
    xs = recipe_subjects(rng, 3, 500, 50, 8, smooth_sigma=5.0, dtype=np.float32)
    save_trace("em_smooth_f32", xs, 8, 3, 5, srm, reference, SerialCommunicator,
               SubjectData, naive=False)

    # tolerance stop (test_srm.py:269-274 pattern)
    rng = np.random.default_rng(3)
    xs = recipe_subjects(rng, 2, 20, 10, 2)
    model = srm.fit([SubjectData(f"s{i}", x) for i, x in enumerate(xs)],
                    srm.SrmConfig(k=2, iterations=50, seed=1, tolerance=1e-8),
                    SerialCommunicator())
    np.savez_compressed(OUT / "tolerance.npz", X0=xs[0], X1=xs[1],
                        n_iter=len(model.objective_trace), S=model.S,
                        W0=model.W[0], W1=model.W[1], rho2=np.array(model.rho2))
    print("wrote tolerance.npz")


if __name__ == "__main__":
    main()
