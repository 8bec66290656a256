"""The CPU oracle (oracle/srm_oracle.py) pinned to the reference's own outputs.

tests/golden/*.npz were produced by tests/golden/make_golden.py, which runs
the real reference package (factorfit) on seeded inputs.  These tests need
no GPU: they prove the restatement reproduces the reference before it is
used as the checker of the CUDA path.
"""

import numpy as np
import pytest

from conftest import golden_subjects, load_golden, nrel
from oracle import srm_oracle as orc


def test_spd_inverse_matches_reference():
    g = load_golden("kernels")
    for j in range(5):
        out = orc.chol_inverse(g[f"spd_in{j}"])
        assert np.array_equal(out, g[f"spd_out{j}"])
    assert np.array_equal(orc.chol_inverse(g["spd_ill_in"]), g["spd_ill_out"])


def test_spd_inverse_pivot():
    g = load_golden("kernels")
    with pytest.raises(orc.OracleError) as ei:
        orc.chol_inverse(g["spd_bad_in"])
    assert ei.value.kind == "DefinitenessError"
    assert ei.value.pivot == int(g["spd_bad_pivot"]) == 3


def test_polar_matches_reference():
    g = load_golden("kernels")
    for j in range(4):
        assert np.array_equal(orc.orthogonal_polar(g[f"polar_in{j}"]), g[f"polar_out{j}"])


def test_polar_rank_error():
    with pytest.raises(orc.OracleError) as ei:
        orc.orthogonal_polar(np.zeros((6, 2)))
    assert ei.value.kind == "RankError"


def test_trace_and_demean():
    g = load_golden("kernels")
    assert orc.sum_of_squares(g["tata_in"]) == float(g["tata_out"])
    for suffix in ("", "2"):
        xh, mu = orc.center_rows(g[f"demean_in{suffix}"])
        assert np.array_equal(xh, g[f"demean_xhat{suffix}"])
        assert np.array_equal(mu, g[f"demean_mu{suffix}"])


def test_init_subject_matches_reference():
    g = load_golden("kernels")
    for j in range(4):
        v, k, seed, idx = (int(x) for x in g[f"init_args{j}"])
        w, rho2 = orc.initial_mapping(v, k, seed, idx)
        assert rho2 == 1.0
        assert np.array_equal(w, g[f"init_W{j}"])


def test_single_steps_match_reference():
    g = load_golden("steps")
    ws = [g[f"W{i}"] for i in range(3)]
    xs = [g[f"Xhat{i}"] for i in range(3)]
    rho2 = list(g["rho2"])
    terms = [orc.local_term(w, r, x) for w, r, x in zip(ws, rho2, xs)]
    for i in range(3):
        assert np.array_equal(terms[i], g[f"local{i}"])
    reduced = sum(terms)
    assert np.array_equal(reduced, g["reduced"])
    s, var = orc.shared_posterior(reduced, g["sigma_s"], float(g["rho0"]))
    assert np.array_equal(s, g["S"]) and np.array_equal(var, g["var_s"])
    sig, tr = orc.shared_covariance(g["sigma_s"], float(g["rho0"]), s)
    assert np.array_equal(sig, g["sigma_new"]) and tr == float(g["trace"])
    for i in range(3):
        w, r = orc.subject_update(xs[i], s, tr)
        assert np.array_equal(w, g[f"mW{i}"]) and r == float(g[f"mrho2_{i}"])
    # Woodbury LL == reference naive LL (SURVEY.md §7 determinant lemma)
    sq = [orc.sum_of_squares(x) for x in xs]
    ll = orc.woodbury_loglik(reduced, float(g["rho0"]), g["sigma_s"], rho2,
                             [x.shape[0] for x in xs], sq, xs[0].shape[1])
    assert abs(ll - float(g["ll_naive"])) <= 1e-10 * abs(float(g["ll_naive"]))
    # Woodbury posterior == naive posterior (test_srm.py:99-107)
    s_n, var_n = orc.naive_posterior(ws, rho2, g["sigma_s"], xs)
    assert np.max(np.abs(s - s_n)) <= 1e-8 and np.max(np.abs(var - var_n)) <= 1e-8


@pytest.mark.parametrize("name", ["em_small", "em_ragged", "em_recipe_f32", "em_smooth_f32"])
def test_em_trace_bit_identical_to_reference(name):
    g = load_golden(name)
    xs = golden_subjects(g)
    out = orc.run_em(xs, int(g["k"]), int(g["iterations"]), seed=int(g["seed"]))
    for it, rec in enumerate(out["iters"]):
        assert np.array_equal(rec["S"], g[f"it{it}_S"])
        assert np.array_equal(rec["sigma_s"], g[f"it{it}_sigma_s"])
        assert np.array_equal(rec["rho2"], g[f"it{it}_rho2"])
        for i in range(len(xs)):
            assert np.array_equal(rec["W"][i], g[f"it{it}_W{i}"])
        if np.isfinite(g[f"it{it}_ll_naive"]):
            ref = float(g[f"it{it}_ll_naive"])
            assert abs(rec["ll"] - ref) <= 1e-10 * abs(ref), (it, rec["ll"], ref)
    assert np.array_equal(out["S"], g["fit_S"])
    assert np.array_equal(out["sigma_s"], g["fit_sigma_s"])
    assert np.array_equal(np.array(out["rho2"]), g["fit_rho2"])
    assert out["rho0"] == float(g["fit_rho0"])
    assert np.array_equal(np.array(out["objective"]), g["fit_objective"])
    for i in range(len(xs)):
        assert np.array_equal(out["W"][i], g[f"fit_W{i}"])
        assert np.array_equal(out["mu"][i], g[f"fit_mu{i}"])


def test_final_loglik_matches_naive():
    g = load_golden("em_small")
    xs = golden_subjects(g)
    out = orc.run_em(xs, int(g["k"]), int(g["iterations"]), seed=int(g["seed"]), record=False)
    xh = [orc.center_rows(x)[0] for x in xs]
    ll = orc.final_loglik(out["W"], out["rho2"], out["sigma_s"], xh)
    ref = float(g["final_ll_naive"])
    assert abs(ll - ref) <= 1e-10 * abs(ref)


def test_log_likelihood_monotone():
    """test_srm.py:247-267 / acceptance criterion 3 on the oracle's Woodbury LL."""
    g = load_golden("em_small")
    out = orc.run_em(golden_subjects(g), int(g["k"]), int(g["iterations"]), seed=int(g["seed"]))
    lls = np.array([r["ll"] for r in out["iters"]])
    assert np.all(np.diff(lls) >= -1e-9)


def test_tolerance_stop_matches_reference():
    g = load_golden("tolerance")
    out = orc.run_em([g["X0"], g["X1"]], 2, 50, seed=1, tolerance=1e-8, record=False)
    assert len(out["objective"]) == int(g["n_iter"])
    assert np.array_equal(out["S"], g["S"])
    assert np.array_equal(out["W"][0], g["W0"]) and np.array_equal(out["W"][1], g["W1"])


def test_flop_model():
    """cli.py:64-72 / acceptance criterion 13."""
    v, t, k = 3000.0, 2201.0, 60.0
    expected = 2.0 * (2.0 * v * t * k) + 2.0 * v * k * k + (2.0 * v * k * k - (2.0 / 3.0) * k ** 3)
    assert orc.flops_per_subject_iteration(3000, 2201, 60) == expected


def test_nrel_helper():
    assert nrel([1.0, 2.0], [1.0, 2.0]) == 0.0


@pytest.mark.parametrize("workers,keep", [(1, True), (3, False)])
def test_em_iterations_bit_identical_to_run_em(workers, keep):
    """The streaming oracle driver used at BASELINE sizes (cached trace_ata and
    W^T Xhat, threads, re-formed Xhat) == run_em, bit for bit, every iteration."""
    g = load_golden("em_ragged")
    xs = golden_subjects(g)
    k, iters, seed = int(g["k"]), int(g["iterations"]), int(g["seed"])
    ref = orc.run_em(xs, k, iters, seed=seed)
    recs = list(orc.em_iterations(xs, k, iters, seed=seed, workers=workers, keep_xhat=keep))
    assert len(recs) == iters
    for a, b in zip(recs, ref["iters"]):
        assert np.array_equal(a["S"], b["S"]) and np.array_equal(a["sigma_s"], b["sigma_s"])
        assert np.array_equal(a["rho2"], b["rho2"]) and a["ll"] == b["ll"] and a["rho0"] == b["rho0"]
        for wa, wb in zip(a["W"], b["W"]):
            assert np.array_equal(wa, wb)
