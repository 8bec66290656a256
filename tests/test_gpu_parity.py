"""CUDA path vs the reference (golden fixtures) and the CPU oracle.

Tolerance (BASELINE.json north_star): per EM iteration, normwise relative
1e-9 for fp64 and 1e-4 for fp32 inputs, on S, every W_i, rho^2, Sigma_s and
the log-likelihood.  Per-iteration states come from fits of 1..N iterations
(the reference's own test_srm.py:231-245 pattern).
"""

import numpy as np
import pytest

from conftest import golden_subjects, load_golden, nrel
from oracle import srm_oracle as orc

pytestmark = pytest.mark.gpu

TOL64 = 1e-9
TOL32 = 1e-4


@pytest.fixture(scope="module")
def srm():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_1608_04647_b200 import srm as mod

    return mod


def _subjects(srm, xs):
    return [srm.SubjectData(f"s{i}", x) for i, x in enumerate(xs)]


def _check_model(model, ref_S, ref_sigma, ref_rho2, ref_W, tol, what=""):
    assert nrel(model.S, ref_S) <= tol, (what, "S", nrel(model.S, ref_S))
    assert nrel(model.sigma_s, ref_sigma) <= tol, (what, "sigma", nrel(model.sigma_s, ref_sigma))
    assert nrel(model.rho2, ref_rho2) <= tol, (what, "rho2", nrel(model.rho2, ref_rho2))
    for i, w in enumerate(ref_W):
        assert nrel(model.W[i], w) <= tol, (what, "W", i, nrel(model.W[i], w))


@pytest.mark.parametrize("name", ["em_small", "em_ragged", "em_recipe_f32", "em_smooth_f32"])
def test_fit_every_iteration_matches_reference(srm, name):
    g = load_golden(name)
    xs = golden_subjects(g)
    k, iters, seed = int(g["k"]), int(g["iterations"]), int(g["seed"])
    tol = TOL64 if xs[0].dtype == np.float64 else TOL32
    for n in range(1, iters + 1):
        m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=k, iterations=n, seed=seed))
        it = n - 1
        _check_model(m, g[f"it{it}_S"], g[f"it{it}_sigma_s"], g[f"it{it}_rho2"],
                     [g[f"it{it}_W{i}"] for i in range(len(xs))], tol, f"{name} it{it}")
        # LL of the parameters entering each iteration vs the reference naive LL
        for j in range(n):
            ref = float(g[f"it{j}_ll_naive"])
            if np.isfinite(ref):
                assert abs(m.log_likelihood[j] - ref) <= TOL64 * abs(ref), (name, j)
        # orthogonality after every M-step (acceptance criterion 4)
        for w in m.W:
            assert np.max(np.abs(w.T @ w - np.eye(k))) <= 1e-8
    assert nrel(m.objective_trace, g["fit_objective"]) <= tol
    assert abs(m.rho0 - float(g["fit_rho0"])) <= tol * abs(float(g["fit_rho0"]))
    for i in range(len(xs)):
        assert nrel(m.mu[i], g[f"fit_mu{i}"]) <= tol or np.max(np.abs(m.mu[i] - g[f"fit_mu{i}"])) <= 1e-12


def test_tolerance_stop(srm):
    g = load_golden("tolerance")
    m = srm.fit(_subjects(srm, [g["X0"], g["X1"]]), srm.SrmConfig(k=2, iterations=50, seed=1, tolerance=1e-8))
    assert len(m.objective_trace) == int(g["n_iter"])
    assert nrel(m.S, g["S"]) <= TOL64


def test_recipe_vs_oracle_moderate(srm):
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(5, 2500, 160, 20, seed=11)
    ref = orc.run_em(xs, 20, 6, seed=0)
    for n in (1, 3, 6):
        m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=20, iterations=n, seed=0))
        r = ref["iters"][n - 1]
        _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL64, f"recipe it{n-1}")
        for j in range(n):
            assert abs(m.log_likelihood[j] - ref["iters"][j]["ll"]) <= TOL64 * abs(ref["iters"][j]["ll"])


def test_cfg1_full_size_vs_oracle(srm):
    """BASELINE cfg 1 (10 x 5000 x 500, K=50, fp64, 10 iterations) at parity."""
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(10, 5000, 500, 50, seed=1)
    ref = orc.run_em(xs, 50, 10, seed=0)
    m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=50, iterations=10, seed=0))
    r = ref["iters"][-1]
    _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL64, "cfg1")
    lls = np.array(m.log_likelihood)
    ref_ll = np.array([x["ll"] for x in ref["iters"]])
    assert np.max(np.abs(lls - ref_ll) / np.abs(ref_ll)) <= TOL64
    assert np.all(np.diff(lls) >= -1e-9 * np.abs(lls[1:]))


# --------------------------------------------------------------------------
# step-function API (srm.py:94-155) vs golden
# --------------------------------------------------------------------------

def test_steps_match_reference(srm):
    g = load_golden("steps")
    ws = [g[f"W{i}"] for i in range(3)]
    xs = [g[f"Xhat{i}"] for i in range(3)]
    for i in range(3):
        assert nrel(srm.e_step_local(ws[i], float(g["rho2"][i]), xs[i]), g[f"local{i}"]) <= 1e-13
    S, var = srm.e_step_global(g["reduced"], g["sigma_s"], float(g["rho0"]))
    assert nrel(S, g["S"]) <= TOL64 and nrel(var, g["var_s"]) <= TOL64
    sig, tr = srm.update_sigma_s(g["sigma_s"], float(g["rho0"]), g["S"])
    assert nrel(sig, g["sigma_new"]) <= TOL64 and abs(tr - float(g["trace"])) <= TOL64 * abs(float(g["trace"]))
    for i in range(3):
        w, r = srm.m_step_subject(xs[i], g["S"], float(g["trace"]))
        assert nrel(w, g[f"mW{i}"]) <= TOL64
        assert abs(r - float(g[f"mrho2_{i}"])) <= TOL64 * abs(float(g[f"mrho2_{i}"]))


def test_demean_and_init_match_reference(srm):
    g = load_golden("kernels")
    xh, mu = srm.demean(g["demean_in"])
    assert np.array_equal(xh, g["demean_xhat"]) and np.array_equal(mu, g["demean_mu"])
    xh, mu = srm.demean(g["demean_in2"])
    assert np.max(np.abs(xh - g["demean_xhat2"])) <= 1e-12 and np.max(np.abs(mu - g["demean_mu2"])) <= 1e-12
    for j in range(4):
        v, k, seed, idx = (int(x) for x in g[f"init_args{j}"])
        w, rho2 = srm.init_subject(v, srm.SrmConfig(k=k, seed=seed), idx)
        assert rho2 == 1.0
        assert nrel(w, g[f"init_W{j}"]) <= 1e-12, (j, nrel(w, g[f"init_W{j}"]))


def test_errors(srm):
    from paper_1608_04647_b200.errors import (DefinitenessError, InvalidInputError, RankError,
                                              ShapeError, ConfigError)

    rng = np.random.default_rng(8)
    with pytest.raises(RankError):
        srm.m_step_subject(rng.standard_normal((6, 4)), np.zeros((2, 4)), 1.0)
    with pytest.raises(DefinitenessError) as ei:
        srm.e_step_global(np.zeros((3, 4)), np.zeros((3, 3)), 1.0)
    assert ei.value.pivot == 0
    x = rng.standard_normal((20, 8))
    x[3, 2] = np.nan
    with pytest.raises(InvalidInputError):
        srm.fit([srm.SubjectData("a", x)], srm.SrmConfig(k=2, iterations=2))
    with pytest.raises(ShapeError):
        srm.fit([srm.SubjectData("a", np.zeros((5, 4))), srm.SubjectData("b", np.zeros((5, 6)))],
                srm.SrmConfig(k=2))
    with pytest.raises(ShapeError):
        srm.init_subject(2, srm.SrmConfig(k=3), 0)
    with pytest.raises(ConfigError):
        srm.fit([], srm.SrmConfig(k=2))


def test_projection(srm):
    g = load_golden("em_small")
    xs = golden_subjects(g)
    m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=4, iterations=5, seed=0))
    assert np.max(np.abs(srm.project(m, 0, m.mu[0]))) == 0.0
    x = xs[1][:, 3]
    z = srm.project(m, 1, x)
    assert nrel(z, m.W[1].T @ (x - m.mu[1])) <= 1e-13
    once = srm.map_between(m, 0, 0, xs[0][:, 0])
    twice = srm.map_between(m, 0, 0, once)
    assert np.max(np.abs(twice - once)) <= 1e-10
    with pytest.raises(IndexError):
        srm.project(m, 7, np.zeros(60))


@pytest.mark.parametrize("name", ["em_small", "em_ragged", "em_recipe_f32"])
@pytest.mark.parametrize("algorithm", ["stream", "gram"])
def test_algorithms_agree_with_reference(srm, name, algorithm):
    g = load_golden(name)
    xs = golden_subjects(g)
    k, iters, seed = int(g["k"]), int(g["iterations"]), int(g["seed"])
    tol = TOL64 if xs[0].dtype == np.float64 else TOL32
    for n in (1, 2, iters):
        m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=k, iterations=n, seed=seed), algorithm=algorithm)
        it = n - 1
        _check_model(m, g[f"it{it}_S"], g[f"it{it}_sigma_s"], g[f"it{it}_rho2"],
                     [g[f"it{it}_W{i}"] for i in range(len(xs))], tol, f"{name} {algorithm} it{it}")


def test_gram_cfg1_full_size_vs_oracle(srm):
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(10, 5000, 500, 50, seed=1)
    ref = orc.run_em(xs, 50, 10, seed=0)
    m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=50, iterations=10, seed=0), algorithm="gram")
    r = ref["iters"][-1]
    _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL64, "cfg1 gram")
    ref_ll = np.array([x["ll"] for x in ref["iters"]])
    assert np.max(np.abs(np.array(m.log_likelihood) - ref_ll) / np.abs(ref_ll)) <= TOL64


@pytest.mark.parametrize("name", ["em_recipe_f32", "em_smooth_f32"])
def test_tensor_core_fp32_path(srm, name):
    """fp32 X-hat through the tcgen05 3xTF32 streaming kernels, every iteration within 1e-4."""
    g = load_golden(name)
    xs = golden_subjects(g)
    k, iters, seed = int(g["k"]), int(g["iterations"]), int(g["seed"])
    engines = []
    for n in range(1, iters + 1):
        m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=k, iterations=n, seed=seed), algorithm="stream",
                    tensor_cores=True, engine_out=engines)
        assert engines[-1].tc, "tensor-core path not selected"
        it = n - 1
        _check_model(m, g[f"it{it}_S"], g[f"it{it}_sigma_s"], g[f"it{it}_rho2"],
                     [g[f"it{it}_W{i}"] for i in range(len(xs))], TOL32, f"{name} tc it{it}")
    # the split-precision error is ~1e-6: far inside the fp32 tolerance
    assert nrel(m.S, g[f"it{iters - 1}_S"]) <= 1e-5


def test_tensor_core_fp32_recipe_vs_oracle(srm):
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(4, 3000, 400, 100, seed=21, dtype="f32")
    ref = orc.run_em(xs, 100, 4, seed=0)
    for n in (1, 4):
        m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=100, iterations=n, seed=0), algorithm="stream",
                    tensor_cores=True)
        r = ref["iters"][n - 1]
        _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL32, f"tc recipe it{n - 1}")


def _gram_pair(xs):
    """X_i^T X_i of the demeaned subjects from the fp64 DMMA and the int8-sliced kernels."""
    import torch

    from paper_1608_04647_b200 import _lib
    from paper_1608_04647_b200.engine import SrmEngine

    T = xs[0].shape[1]
    out = []
    for i8 in (False, True):
        eng = SrmEngine([x.shape[0] for x in xs], T, 4, 1, gram=True, gram_i8=i8)
        assert eng.gram_i8 == i8, "int8 Gram flag not effective"
        eng.load(xs)
        eng.prepare_gram()
        torch.cuda.synchronize()
        eng.raise_status()
        full = eng.region(_lib.R_GRAM, torch.float64).view(len(xs), eng.ldx, eng.ldx)
        if i8:  # the padded TRs (T..ldx): zeros, also where a tile's N was trimmed to T
            assert torch.count_nonzero(full[:, T:, :]) == 0 and torch.count_nonzero(full[:, :, T:]) == 0
        out.append(full[:, :T, :T].cpu().numpy())
        eng.close()
    return out


@pytest.mark.parametrize("case", ["recipe", "ragged_t300", "heavy_tails", "long_v", "pipelined"])
def test_int8_gram_matches_fp64(srm, case):
    """The int8-sliced X^T X (7 slices, exact int32 sums) vs fp64 DMMA and numpy."""
    from paper_1608_04647_b200.data import recipe_numpy

    rng = np.random.default_rng(7)
    tol = 1e-13
    if case == "recipe":
        xs = recipe_numpy(3, 2000, 256, 10, seed=4)[0]
    elif case == "ragged_t300":  # T not a multiple of 128 (partial tiles), ragged V
        xs = [rng.standard_normal((v, 300)) for v in (1000, 777, 1531)]
    elif case == "heavy_tails":  # Student t (2 dof): column max / rms ~ 10-100
        xs = [rng.standard_t(2, size=(3000, 200)) for _ in range(2)]
        tol = 1e-11
    elif case == "pipelined":  # T = 1000: 36 tiles per subject, Gram batches of 4 behind the side-stream slicing
        xs = [rng.standard_normal((v, 1000)) for v in (700, 911, 640, 1003, 777, 850, 690, 1200, 530, 960)]
    else:  # > 65536 voxels: the int32 accumulators are flushed per 65536-voxel chunk
        xs = [rng.standard_normal((70000, 64))]
    g_dmma, g_i8 = _gram_pair(xs)
    for i, x in enumerate(xs):
        xh = x - x.mean(axis=1, keepdims=True)
        ref = xh.T @ xh
        assert nrel(g_dmma[i], ref) <= 1e-14, (case, i, "dmma", nrel(g_dmma[i], ref))
        assert nrel(g_i8[i], ref) <= tol, (case, i, "i8", nrel(g_i8[i], ref))
        assert np.array_equal(g_i8[i], g_i8[i].T)


def test_int8_gram_fit_matches_oracle(srm):
    """Full fit through the int8-sliced Gram (the default Gram path for fp64) vs the oracle."""
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(6, 4000, 384, 40, seed=9)
    ref = orc.run_em(xs, 40, 6, seed=0)
    for i8 in (True, False):
        engines = []
        m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=40, iterations=6, seed=0), algorithm="gram",
                    gram_int8=i8, engine_out=engines)
        assert engines[-1].gram and engines[-1].gram_i8 == i8
        r = ref["iters"][-1]
        _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL64, f"gram i8={i8}")
        ref_ll = np.array([x["ll"] for x in ref["iters"]])
        assert np.max(np.abs(np.array(m.log_likelihood) - ref_ll) / np.abs(ref_ll)) <= TOL64


def test_fit_manifest_streams_sfab(srm, tmp_path):
    """SFAB files -> pinned slots -> device (data_io.fit_manifest) == srm.fit on the same arrays."""
    from paper_1608_04647_b200 import data_io
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(5, 900, 64, 6, seed=13)
    xs = [x[: 900 - 41 * i] for i, x in enumerate(xs)]  # ragged V; 5 subjects > 3 read-ahead slots
    entries = []
    for i, x in enumerate(xs):
        p = tmp_path / f"s{i}.sfab"
        data_io.save_matrix(p, x)
        entries.append(data_io.ManifestEntry(f"s{i}", p))
    man = tmp_path / "m.json"
    data_io.write_manifest(man, data_io.Manifest("t", entries))
    cfg = srm.SrmConfig(k=6, iterations=4, seed=3)
    a = data_io.fit_manifest(man, cfg)
    b = srm.fit([srm.SubjectData(f"s{i}", x) for i, x in enumerate(xs)], cfg)
    assert a.subject_ids == b.subject_ids
    assert np.array_equal(a.S, b.S) and np.array_equal(a.sigma_s, b.sigma_s)
    for wa, wb in zip(a.W, b.W):
        assert np.array_equal(wa, wb)
    assert a.rho2 == b.rho2


def test_int8_gram_k72_two_feature_halves(srm):
    """K = 72 (kp > 64): the int8 row GEMMs (B = S G / 2, final W) in two 64-feature halves."""
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(3, 2500, 256, 72, seed=15)
    ref = orc.run_em(xs, 72, 3, seed=2)
    engines = []
    m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=72, iterations=3, seed=2), algorithm="gram",
                engine_out=engines)
    assert engines[-1].gram_i8
    r = ref["iters"][-1]
    _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL64, "gram i8 k=72")


def test_int8_gram_fp32_four_slices(srm):
    """fp32 X-hat on the int8 Gram path: 4 slices per value (2^-27 of the column max)."""
    from paper_1608_04647_b200 import _lib
    from paper_1608_04647_b200.data import recipe_numpy
    from paper_1608_04647_b200.engine import SrmEngine
    import torch

    xs, _, _ = recipe_numpy(3, 3000, 300, 20, seed=8, dtype="f32")
    eng = SrmEngine([x.shape[0] for x in xs], 300, 20, 1, storage="f32", gram=True, gram_i8=True)
    assert eng.gram_i8 and not eng.tc
    eng.load(xs)
    eng.prepare_gram()
    torch.cuda.synchronize()
    eng.raise_status()
    g = eng.region(_lib.R_GRAM, torch.float64).view(3, eng.ldx, eng.ldx)[:, :300, :300].cpu().numpy()
    xh = [eng.xhat[eng.subject_rows(i)][:, :300].double().cpu().numpy() for i in range(3)]
    eng.close()
    for i in range(3):
        ref = xh[i].T @ xh[i]
        assert nrel(g[i], ref) <= 1e-6, (i, nrel(g[i], ref))
    # and a full fit at the fp32 tolerance
    ref = orc.run_em(xs, 20, 4, seed=1)
    engines = []
    m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=20, iterations=4, seed=1), algorithm="gram",
                engine_out=engines)
    assert engines[-1].gram_i8
    r = ref["iters"][-1]
    _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL32, "gram i8 fp32")


def test_int8_gram_fp32_large_k_ragged(srm):
    """fp32, K = 100 (two 64-feature halves, fp32 polar per iteration, exact final polar),
    ragged V and T = 330 (partial 128-TR tiles) on the int8 Gram path."""
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(3, 2600, 330, 100, seed=23, dtype="f32")
    xs = [x[: 2600 - 97 * i] for i, x in enumerate(xs)]
    ref = orc.run_em(xs, 100, 3, seed=4)
    engines = []
    m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=100, iterations=3, seed=4), algorithm="gram",
                engine_out=engines)
    assert engines[-1].gram_i8
    r = ref["iters"][-1]
    _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL32, "gram i8 fp32 k=100")
    for w in m.W:  # the exact final polar (a subject this small keeps every slice pair of its
        # Gram); W = Xhat R from the pairs s + s' <= 4 of fp32 X-hat's slices: ~1e-10
        assert np.max(np.abs(w.T @ w - np.eye(100))) <= 1e-9


def test_init_overlap_is_bit_identical(srm):
    """The initial mapping run batch by batch during the upload == run once after it."""
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(9, 1200, 160, 12, seed=31)
    cfg = srm.SrmConfig(k=12, iterations=3, seed=6)
    for algorithm in ("gram", "stream"):
        a = srm.fit(_subjects(srm, xs), cfg, algorithm=algorithm, init_overlap=True)
        b = srm.fit(_subjects(srm, xs), cfg, algorithm=algorithm, init_overlap=False)
        assert np.array_equal(a.S, b.S) and np.array_equal(a.sigma_s, b.sigma_s), algorithm
        for wa, wb in zip(a.W, b.W):
            assert np.array_equal(wa, wb), algorithm


def test_batched_finalize_readback_is_bit_identical(srm):
    """W formed and read back in subject batches (srm_finalize_range) == one srm_finalize."""
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(7, 900, 130, 10, seed=5)
    xs[3] = xs[3][:517]  # ragged: a partial 128-voxel tile inside a batch
    cfg = srm.SrmConfig(k=10, iterations=2, seed=2)
    for algorithm in ("gram", "stream"):
        a = srm.fit(_subjects(srm, xs), cfg, algorithm=algorithm)
        b = srm.fit(_subjects(srm, xs), cfg, algorithm=algorithm, keep_on_device=True)
        for wa, wb in zip(a.W, b.W):
            assert np.array_equal(wa, wb.cpu().numpy()), algorithm


def test_eager_two_lane_iteration_matches_graph(srm):
    """srm_e_step / srm_m_step issued eagerly (side-stream stages joined per
    call) == the captured one-iteration graph, bit for bit, on both paths."""
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(6, 800, 140, 9, seed=21)
    cfg = srm.SrmConfig(k=9, iterations=4, seed=3)
    for algorithm in ("gram", "stream"):
        a = srm.fit(_subjects(srm, xs), cfg, algorithm=algorithm, graphs=True)
        b = srm.fit(_subjects(srm, xs), cfg, algorithm=algorithm, graphs=False)
        assert np.array_equal(a.S, b.S) and np.array_equal(a.sigma_s, b.sigma_s), algorithm
        assert a.log_likelihood == b.log_likelihood, algorithm
        for wa, wb in zip(a.W, b.W):
            assert np.array_equal(wa, wb), algorithm



def test_cfg2_full_size_vs_oracle(srm):
    """BASELINE cfg 2 at full size (40 x 30000 x 1000, K=50, fp64) through the
    default path (int8 Gram, int8 B = S G, int8 final W) vs the oracle, every
    one of the first three iterations."""
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(40, 30000, 1000, 50, seed=2)
    ref = orc.run_em(xs, 50, 3, seed=0)
    for n in (1, 3):
        eng = []
        # the path auto picks at the BASELINE's 20 iterations (at 1-3 it would stream)
        m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=50, iterations=n, seed=0), engine_out=eng,
                    algorithm="gram")
        assert eng[0].gram and eng[0].gram_i8
        r = ref["iters"][n - 1]
        _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL64, f"cfg2 it{n - 1}")
        for j in range(n):
            assert abs(m.log_likelihood[j] - ref["iters"][j]["ll"]) <= TOL64 * abs(ref["iters"][j]["ll"])
        for w in m.W:
            assert np.max(np.abs(w.T @ w - np.eye(50))) <= 1e-8


def test_int8_path_extreme_magnitudes(srm):
    """Subjects scaled by 1e40, 1e-40 and 1: the per-column / per-row
    power-of-two scales of the int8 slices span ~2^±133 (G and S G ~2^±270),
    far outside int8 and fp32 range, and the fit still matches the oracle.
    (The polar through A^T A squares |A|: the fp64 range bounds |A| < 1e154,
    a limit the reference's SVD of A does not have.)"""
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(3, 600, 200, 5, seed=17)
    xs = [xs[0] * 1e40, xs[1] * 1e-40, xs[2]]
    ref = orc.run_em(xs, 5, 3, seed=4)
    eng = []
    m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=5, iterations=3, seed=4), algorithm="gram", engine_out=eng)
    assert eng[0].gram_i8
    r = ref["iters"][-1]
    _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL64, "extreme magnitudes")


# --------------------------------------------------------------------------
# BASELINE cfg 3 / 4 / 5 at their full per-subject shapes (V, T, K, fp32
# storage, cfg 4's smoothed W_i).  The oracle cannot run 16 / 256 / 128
# subjects of these sizes in a test, so each case takes the first few
# subjects of the config's seeded recipe (same V, T, K, dtype, recipe) and
# two EM iterations on both device algorithms; the fp32 tolerance applies.
# --------------------------------------------------------------------------

_FULL_SHAPES = {
    # name: (subjects kept, V, T, K, smooth)
    "cfg3": (2, 200000, 2000, 100, None),
    "cfg4": (4, 50000, 1000, 64, 5.0),
    "cfg5": (3, 100000, 1000, 100, None),
}


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4", "cfg5"])
def test_fp32_configs_full_shape_vs_oracle(srm, cfg):
    import torch

    from paper_1608_04647_b200.data import recipe_torch

    n, V, T, K, smooth = _FULL_SHAPES[cfg]
    xd, _, _ = recipe_torch(n, V, T, K, seed=5, smooth=smooth, dtype="f32")
    xs = [x.cpu().numpy() for x in xd]
    del xd
    torch.cuda.empty_cache()
    iters = 2
    ref = orc.run_em(xs, K, iters, seed=0)
    for algorithm in ("gram", "stream"):
        eng = []
        m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=K, iterations=iters, seed=0), algorithm=algorithm,
                    engine_out=eng)
        assert eng[0].gram == (algorithm == "gram"), (cfg, algorithm)
        r = ref["iters"][-1]
        _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL32, f"{cfg} {algorithm}")
        for j in range(iters):
            assert abs(m.log_likelihood[j] - ref["iters"][j]["ll"]) <= TOL32 * abs(ref["iters"][j]["ll"])
        for w in m.W:
            assert np.max(np.abs(w.T @ w - np.eye(K))) <= 1e-8, (cfg, algorithm)
        del m
        torch.cuda.empty_cache()


def _sg_fit(srm, xs, k, per_tile, monkeypatch):
    monkeypatch.setenv("SRM_B200_SG_PER_TILE", "1" if per_tile else "0")
    eng = []
    m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=k, iterations=3, seed=2), algorithm="gram", engine_out=eng)
    assert eng[0].gram_i8
    return m


@pytest.mark.parametrize("k", [20, 72])
def test_stream_k_sg_bit_identical_to_per_tile(srm, monkeypatch, k):
    """B = S G / 2 stream-K (tiles cut between persistent CTAs, the parts
    joined in int32) against the per-tile grid: the same fit bit for bit.
    10 subjects x T = 2000 make ~70 k-blocks per CTA, so most CTAs split a
    tile; K = 72 adds the second 64-feature half."""
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(10, 400, 2000, k, seed=8)
    a = _sg_fit(srm, xs, k, False, monkeypatch)
    b = _sg_fit(srm, xs, k, True, monkeypatch)
    assert np.array_equal(a.S, b.S) and np.array_equal(a.sigma_s, b.sigma_s)
    assert np.array_equal(a.rho2, b.rho2) and a.log_likelihood == b.log_likelihood
    for wa, wb in zip(a.W, b.W):
        assert np.array_equal(wa, wb)
    ref = orc.run_em(xs, k, 3, seed=2)
    r = ref["iters"][-1]
    _check_model(a, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL64, f"stream-K k={k}")


# --------------------------------------------------------------------------
# polar conditioning: the Gram-route transform (A^T A)^{-1/2} vs the exact
# route (TSQR + SVD of A, SRM_FLAG_EXACT_POLAR) the fit falls back to
# --------------------------------------------------------------------------

def _lowrank_subjects(noise, seed=0, V=300, T=60, K=5, N=3):
    """X_i = W_i S + noise, with the last of K shared components absent: A_i =
    Xhat_i S^T / 2 has cond ~ (1 / noise)^2 (2e5 at noise 1e-3, 2e9 at 1e-5;
    the reference raises RankError at 1e-7)."""
    rng = np.random.default_rng(seed)
    s = rng.standard_normal((K, T))
    s[-1] = 0.0
    xs = []
    for _ in range(N):
        w = np.linalg.qr(rng.standard_normal((V, K)))[0]
        xs.append(w @ s + noise * rng.standard_normal((V, T)))
    return xs


@pytest.mark.parametrize("name", ["em_small", "em_ragged", "em_recipe_f32"])
def test_exact_polar_route_every_iteration(srm, name):
    """exact_polar=True (TSQR + one-sided Jacobi SVD of every A_i) against the
    reference's golden fit at every iteration."""
    g = load_golden(name)
    xs = golden_subjects(g)
    k, iters, seed = int(g["k"]), int(g["iterations"]), int(g["seed"])
    tol = TOL64 if xs[0].dtype == np.float64 else TOL32
    for n in range(1, iters + 1):
        eng = []
        m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=k, iterations=n, seed=seed), exact_polar=True,
                    engine_out=eng)
        assert eng[-1].exact_polar and not eng[-1].gram
        it = n - 1
        _check_model(m, g[f"it{it}_S"], g[f"it{it}_sigma_s"], g[f"it{it}_rho2"],
                     [g[f"it{it}_W{i}"] for i in range(len(xs))], tol, f"{name} exact it{it}")
        for w in m.W:
            assert np.max(np.abs(w.T @ w - np.eye(k))) <= 1e-8


@pytest.mark.parametrize("algorithm", ["gram", "stream"])
def test_ill_conditioned_fit_falls_back_to_exact_polar(srm, algorithm):
    """cond(A_i) ~ 2e3: beyond the Gram route (c / lambda_min > 1e5 raises the
    device warning), inside the reference's rank threshold -- the fit is redone
    on the exact route and matches the oracle at every iteration, every array
    at the fp64 tolerance."""
    xs = _lowrank_subjects(1e-2)
    ref = orc.run_em(xs, 5, 6, seed=0)
    for n in range(1, 7):
        eng = []
        m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=5, iterations=n, seed=0), algorithm=algorithm,
                    engine_out=eng)
        assert len(eng) == 2 and not eng[0].exact_polar and eng[1].exact_polar, (algorithm, n)
        r = ref["iters"][n - 1]
        _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL64, f"lowrank {algorithm} it{n - 1}")
        for w in m.W:
            assert np.max(np.abs(w.T @ w - np.eye(5))) <= 1e-12


@pytest.mark.parametrize("algorithm", ["gram", "stream"])
def test_very_ill_conditioned_fit_at_its_conditioning(srm, algorithm):
    """cond(A_i) ~ 2e5 and rho^2 ~ 1e-6 (a 1e-4 cancellation in srm.py:153-154):
    S at the fp64 tolerance; W_i, rho^2 and Sigma_s within what their own
    conditioning allows any two roundings to differ (cond(A_i) x 1e-13 for
    W_i -- the perturbation bound of the polar factor -- 1e-6 for rho^2, and
    Sigma_s through rho0 = sum 1 / rho_i^2)."""
    xs = _lowrank_subjects(1e-3)
    ref = orc.run_em(xs, 5, 6, seed=0)
    xh = [orc.center_rows(x)[0] for x in xs]
    for n in range(1, 7):
        eng = []
        m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=5, iterations=n, seed=0), algorithm=algorithm,
                    engine_out=eng)
        assert len(eng) == 2 and not eng[0].exact_polar and eng[1].exact_polar, (algorithm, n)
        r = ref["iters"][n - 1]
        what = f"lowrank {algorithm} it{n - 1}"
        assert nrel(m.S, r["S"]) <= TOL64, (what, nrel(m.S, r["S"]))
        assert nrel(m.sigma_s, r["sigma_s"]) <= 1e-7, what
        assert nrel(m.rho2, r["rho2"]) <= 1e-6, what
        # the polar factor's own condition number is cond(A_i): S agrees to
        # ~1e-14, so any two implementations differ in W_i by ~cond(A_i) 1e-14
        for i, w in enumerate(r["W"]):
            cond = np.linalg.cond(0.5 * (xh[i] @ r["S"].T))
            assert nrel(m.W[i], w) <= max(TOL64, 1e-13 * cond), (what, i, nrel(m.W[i], w), cond)
        for w in m.W:
            assert np.max(np.abs(w.T @ w - np.eye(5))) <= 1e-10


def test_nearly_singular_fit_no_spurious_rank_error(srm):
    """cond(A_i) ~ 2e9 (sigma ratio 5e-10, above the reference's 1e-12): the
    reference fits it, so must we; S agrees to ~eps cond."""
    xs = _lowrank_subjects(1e-5)
    ref = orc.run_em(xs, 5, 4, seed=0)
    m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=5, iterations=4, seed=0))
    assert nrel(m.S, ref["S"]) <= 1e-5
    # rho^2 ~ 3e-9 is a 1e-9-relative cancellation of |Xhat|^2 + T tr(Sigma) - 2 cross
    # (srm.py:153-154): any change of rounding moves it by ~10%, the reference's own value included
    assert nrel(m.rho2, ref["rho2"]) <= 0.3


@pytest.mark.parametrize("algorithm", ["gram", "stream"])
def test_rank_deficient_fit_raises_like_reference(srm, algorithm):
    """noise 1e-7: the reference's gesdd polar raises RankError in the M-step."""
    from paper_1608_04647_b200.errors import RankError

    xs = _lowrank_subjects(1e-7)
    with pytest.raises(orc.OracleError, match="RankError"):
        orc.run_em(xs, 5, 6, seed=0)
    with pytest.raises(RankError):
        srm.fit(_subjects(srm, xs), srm.SrmConfig(k=5, iterations=6, seed=0), algorithm=algorithm)


# --------------------------------------------------------------------------
# transforms over blocks of volumes (srm.py:330-338)
# --------------------------------------------------------------------------

def test_project_and_map_between_blocks(srm):
    g = load_golden("em_ragged")
    xs = golden_subjects(g)
    m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=int(g["k"]), iterations=4, seed=0))
    rng = np.random.default_rng(21)
    for i, j in [(0, 1), (2, 0), (1, 1)]:
        X = xs[i][:, :17] + rng.standard_normal((xs[i].shape[0], 17))
        ref_z = m.W[i].T @ (X - m.mu[i][:, None])
        z = srm.project_batch(m, i, X)
        assert z.shape == ref_z.shape and nrel(z, ref_z) <= 1e-14
        ref_y = m.W[j] @ ref_z + m.mu[j][:, None]
        y = srm.map_between_batch(m, i, j, X)
        assert y.shape == (xs[j].shape[0], 17) and nrel(y, ref_y) <= 1e-14
        # the single-volume API is the one-column case
        for c in (0, 16):
            assert nrel(srm.project(m, i, X[:, c]), ref_z[:, c]) <= 1e-14
            assert nrel(srm.map_between(m, i, j, X[:, c]), ref_y[:, c]) <= 1e-14
    # the mean of a subject projects to exactly zero (test_srm.py:343-345), in every column
    z = srm.project_batch(m, 1, np.repeat(m.mu[1][:, None], 5, axis=1))
    assert np.max(np.abs(z)) == 0.0
    # fp32 volumes are widened to fp64 before the centering, as np.asarray(x, float64)
    X32 = xs[0][:, :9].astype(np.float32)
    ref = m.W[0].T @ (X32.astype(np.float64) - m.mu[0][:, None])
    assert nrel(srm.project_batch(m, 0, X32), ref) <= 1e-14
    # a long block (T' = 700 > one 128-column tile, > 64-column GEMM tiles)
    X = rng.standard_normal((xs[2].shape[0], 700))
    y = srm.map_between_batch(m, 2, 3, X)
    assert nrel(y, m.W[3] @ (m.W[2].T @ (X - m.mu[2][:, None])) + m.mu[3][:, None]) <= 1e-14
    with pytest.raises(IndexError):
        srm.project_batch(m, 4, X)
    with pytest.raises(IndexError):
        srm.map_between_batch(m, 0, -5, xs[0])
    from paper_1608_04647_b200.errors import ShapeError
    with pytest.raises(ShapeError):
        srm.project_batch(m, 0, np.zeros((3, 2)))


def test_transform_reference_cases(srm):
    """test_srm.py:334-367 restated: the square mapping round-trips, the tall
    mapping is idempotent."""
    from paper_1608_04647_b200 import kernels

    rng = np.random.default_rng(15)
    k = 4
    w_true = kernels.polar_orthogonal(rng.standard_normal((k, k)))
    X = w_true @ rng.standard_normal((k, 9))
    model = srm.fit([srm.SubjectData("s0", X)], srm.SrmConfig(k=k, iterations=3, seed=4))
    x = rng.standard_normal(k)
    assert np.max(np.abs(srm.map_between(model, 0, 0, x) - x)) <= 1e-10
    g = load_golden("em_small")
    m = srm.fit(_subjects(srm, golden_subjects(g)), srm.SrmConfig(k=int(g["k"]), iterations=5, seed=2))
    x = rng.standard_normal(m.W[0].shape[0])
    once = srm.map_between(m, 0, 0, x)
    assert np.max(np.abs(srm.map_between(m, 0, 0, once) - once)) <= 1e-10


@pytest.mark.parametrize("dtype,K", [("f64", 50), ("f32", 100), ("f32", 20), ("f64", 100)])
def test_int8_init_term_matches_dmma(srm, dtype, K):
    """The initial E-step term W_0^T Xhat = M_0^T (G^T Xhat) with G^T Xhat from
    the int8 slices of the draw and of X-hat (int8 Gram plans) against the
    fp64 DMMA contraction (fp64 Gram plans), per subject; the int8 plan is
    initialised before any srm_prepare_gram call (it slices X-hat itself).
    K > 64 also forms the draw's G^T G (for M_0) from its slices.  fp32 X-hat:
    the slice pairs s + s' <= 3 only (~1e-7 of the term)."""
    import torch

    from paper_1608_04647_b200.data import recipe_numpy
    from paper_1608_04647_b200.engine import SrmEngine

    xs, _, _ = recipe_numpy(3, 2000, 300, K, seed=41, dtype=dtype)
    xs[1] = xs[1][:1531]  # ragged V: a partial 32-voxel block
    terms = []
    for i8 in (True, False):
        eng = SrmEngine([x.shape[0] for x in xs], 300, K, 2, storage=dtype, gram=True, gram_i8=i8)
        assert eng.gram_i8 == i8
        eng.load(xs)
        eng.init_mapping(7, 0)
        torch.cuda.synchronize()
        eng.raise_status()
        t = eng.terms[:, : eng.kp * eng.ldx].view(-1, eng.kp, eng.ldx)[:, :K, :300].cpu().numpy()
        terms.append(t)
        eng.close()
    tol = 1e-13 if dtype == "f64" else 5e-7  # four fp32 slices, pairs s + s' <= 3
    for j in range(3):
        assert nrel(terms[0][j], terms[1][j]) <= tol, (j, nrel(terms[0][j], terms[1][j]))


@pytest.mark.parametrize("dtype,T,V", [("f64", 1000, 1500), ("f32", 300, 1500), ("f64", 130, 1500),
                                       ("f32", 400, 17000)])
def test_int8_gram_cta_pairs_bit_identical(srm, monkeypatch, dtype, T, V):
    """X^T X from the CTA-pair kernel (tcgen05 cta_group::2, M = 256) equals the
    single-CTA kernel's bit for bit: same slice products, same exact int32 /
    int64 sums, same epilogue; odd and even tile counts, partial tiles; fp32
    subjects of >= 16384 voxels (pass 1 only off the diagonal) beside a
    smaller one (every pair)."""
    import torch

    from paper_1608_04647_b200 import _lib
    from paper_1608_04647_b200.data import recipe_numpy
    from paper_1608_04647_b200.engine import SrmEngine

    xs, _, _ = recipe_numpy(3, V, T, 10, seed=43, dtype=dtype)
    xs[2] = xs[2][:977]
    out = []
    for pairs in ("1", "0"):  # the pair kernel is opt-in (no faster at T = 1000)
        monkeypatch.setenv("SRM_B200_GRAM_PAIRS", pairs)
        eng = SrmEngine([x.shape[0] for x in xs], T, 10, 1, storage=dtype, gram=True, gram_i8=True)
        eng.load(xs)
        eng.prepare_gram()
        torch.cuda.synchronize()
        eng.raise_status()
        g = eng.region(_lib.R_GRAM, torch.float64).view(3, eng.ldx, eng.ldx)[:, :T, :T].cpu().numpy()
        out.append(g)
        eng.close()
    assert np.array_equal(out[0], out[1])
    xh = [x.astype(np.float64) - x.astype(np.float64).mean(axis=1, keepdims=True) for x in xs]
    for i in range(3):
        assert nrel(out[0][i], xh[i].T @ xh[i]) <= (1e-13 if dtype == "f64" else 1e-6)


@pytest.mark.parametrize("dtype,K", [("f64", 50), ("f32", 64), ("f32", 9)])
def test_int8_init_transposed_bit_identical(srm, monkeypatch, dtype, K):
    """kp <= 64: the transposed one-pass init GEMM (M = 128 TRs x N = 64
    features) gives the same G^T Xhat, bit for bit, as the M = 128 feature
    kernel (same exact d-group sums, same epilogue arithmetic)."""
    import torch

    from paper_1608_04647_b200.data import recipe_numpy
    from paper_1608_04647_b200.engine import SrmEngine

    xs, _, _ = recipe_numpy(3, 1700, 260, K, seed=47, dtype=dtype)
    xs[0] = xs[0][:1333]
    out = []
    for nt in ("1", "0"):
        monkeypatch.setenv("SRM_B200_INIT_NT", nt)
        eng = SrmEngine([x.shape[0] for x in xs], 260, K, 2, storage=dtype, gram=True, gram_i8=True)
        eng.load(xs, gram=True)
        eng.init_mapping(3, 0)
        torch.cuda.synchronize()
        eng.raise_status()
        out.append(eng.terms[:, : eng.kp * eng.ldx].cpu().numpy())
        eng.close()
    assert np.array_equal(out[0], out[1])


# --------------------------------------------------------------------------
# K up to 128 (kp 120 / 128: 8 x 8 register sweeps, 64-column apply tiles,
# the L2 Newton-Schulz, the SVD's V in global memory on the exact route)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("K,dtype,algorithm", [(128, "f64", "gram"), (128, "f64", "stream"), (120, "f32", "gram"),
                                              (128, "f32", "stream")])
def test_wide_k_fit_vs_oracle(srm, K, dtype, algorithm):
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(3, 1400, 400, K, seed=53, dtype=dtype)
    xs[1] = xs[1][:1201]
    ref = orc.run_em(xs, K, 3, seed=5)
    tol = TOL64 if dtype == "f64" else TOL32
    for n in (1, 3):
        eng = []
        m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=K, iterations=n, seed=5), algorithm=algorithm,
                    engine_out=eng)
        assert not eng[-1].exact_polar
        r = ref["iters"][n - 1]
        _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], tol, f"K={K} {dtype} {algorithm} it{n - 1}")
        for j in range(n):
            assert abs(m.log_likelihood[j] - ref["iters"][j]["ll"]) <= tol * abs(ref["iters"][j]["ll"])
        # fp32 X-hat on the int8 path: W = Xhat R from the slice pairs s + s' <= 4 (~1e-10)
        orth = 1e-9 if (dtype, algorithm) == ("f32", "gram") else 1e-10
        for w in m.W:
            assert np.max(np.abs(w.T @ w - np.eye(K))) <= orth


def test_wide_k_exact_polar_and_kernels(srm):
    from paper_1608_04647_b200 import kernels
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(2, 900, 300, 128, seed=59)
    ref = orc.run_em(xs, 128, 2, seed=1)
    m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=128, iterations=2, seed=1), exact_polar=True)
    r = ref["iters"][-1]
    _check_model(m, r["S"], r["sigma_s"], r["rho2"], r["W"], TOL64, "K=128 exact")
    rng = np.random.default_rng(61)
    a = rng.standard_normal((3000, 128))
    u, _, vt = np.linalg.svd(a, full_matrices=False)
    assert nrel(kernels.polar_orthogonal(a), u @ vt) <= 1e-12
    c = rng.standard_normal((128, 128))
    spd = c.T @ c + 128 * np.eye(128)
    inv = kernels.spd_inverse(spd)
    assert np.max(np.abs(spd @ inv - np.eye(128))) <= 1e-10 and np.array_equal(inv, inv.T)


def test_step_api_native_pieces(srm):
    """update_sigma_s / m_step_subject compute the symmetrised Sigma, its trace,
    the cross term and trace_ata on the device (srm_sigma_update, srm_dot,
    srm_trace_ata); vs the oracle steps and the non-finite error path."""
    from paper_1608_04647_b200.errors import InvalidInputError

    rng = np.random.default_rng(71)
    k, t, v = 7, 40, 300
    sig = np.cov(rng.standard_normal((k, 3 * k))) + np.eye(k)
    s = rng.standard_normal((k, t))
    ref_sig, ref_tr = orc.shared_covariance(sig, 3.5, s)
    new, tr = srm.update_sigma_s(sig, 3.5, s)
    assert nrel(new, ref_sig) <= 1e-14 and abs(tr - ref_tr) <= 1e-14 * abs(ref_tr) and np.array_equal(new, new.T)
    xh = rng.standard_normal((v, t))
    xh -= xh.mean(axis=1, keepdims=True)
    w_ref, r_ref = orc.subject_update(xh, s, ref_tr)
    w, r = srm.m_step_subject(xh, s, ref_tr)
    assert nrel(w, w_ref) <= 1e-13 and abs(r - r_ref) <= 1e-13 * r_ref
    bad = xh.copy()
    bad[5, 7] = np.inf
    with pytest.raises(InvalidInputError):
        srm.m_step_subject(bad, s, ref_tr)


# --------------------------------------------------------------------------
# seeded random shapes: every path against the oracle at edge sizes
# (K = 1, T = 2, V = K, one subject, T / V / K off every tile multiple)
# --------------------------------------------------------------------------

_EDGE_CASES = [
    # (subjects, V, T, K, dtype, algorithm)
    (1, 40, 2, 1, "f64", "stream"),
    (1, 9, 12, 9, "f64", "gram"),       # V = K: a square polar
    (2, 33, 5, 3, "f64", "gram"),
    (3, 130, 131, 17, "f64", "gram"),   # T = 131: a partial 128-TR tile, K off a multiple of 8
    (3, 257, 33, 12, "f64", "stream"),
    (2, 1001, 257, 65, "f32", "gram"),  # kp = 72 > 64: two 64-feature halves
    (4, 77, 300, 30, "f32", "stream"),
    (2, 500, 97, 31, "f64", "exact"),
    (5, 60, 45, 8, "f32", "gram"),
]


@pytest.mark.parametrize("n,v,t,k,dtype,algorithm", _EDGE_CASES)
def test_edge_shapes_vs_oracle(srm, n, v, t, k, dtype, algorithm):
    rng = np.random.default_rng(1000 + 7 * v + t)
    np_dt = np.float64 if dtype == "f64" else np.float32
    xs = [(rng.standard_normal((v - 3 * j if v - 3 * j >= k else v, t)) * (1 + j)).astype(np_dt) for j in range(n)]
    iters = 4
    ref = orc.run_em(xs, k, iters, seed=3)
    kw = {"exact_polar": True} if algorithm == "exact" else {"algorithm": algorithm}
    tol = TOL64 if dtype == "f64" else TOL32
    states = []
    m = srm.fit(_subjects(srm, xs), srm.SrmConfig(k=k, iterations=iters, seed=3), on_iteration=states.append, **kw)
    states = states[-iters:]  # a fit redone on the exact polar route reports its iterations again
    assert [s.iteration for s in states] == list(range(iters))
    for st, r in zip(states, ref["iters"]):
        what = f"{(n, v, t, k, dtype, algorithm)} it{st.iteration}"
        assert nrel(st.S, r["S"]) <= tol, (what, "S", nrel(st.S, r["S"]))
        assert nrel(st.sigma_s, r["sigma_s"]) <= tol, (what, "sigma")
        assert nrel(st.rho2, r["rho2"]) <= tol, (what, "rho2")
        for w, rw in zip(st.W, r["W"]):
            assert nrel(w, rw) <= tol, (what, "W", nrel(w, rw))
        assert abs(st.log_likelihood - r["ll"]) <= tol * abs(r["ll"]), (what, "ll")
    assert nrel(m.S, ref["S"]) <= tol


@pytest.mark.parametrize("algorithm", ["gram", "stream"])
def test_fewer_trs_than_features_raises_like_reference(srm, algorithm):
    """T < K: S has rank <= T, so A = Xhat S^T / 2 is rank deficient; the
    reference's polar raises RankError in the first M-step (srm.py:148)."""
    from paper_1608_04647_b200.errors import RankError

    rng = np.random.default_rng(77)
    xs = [rng.standard_normal((20, 7))]
    with pytest.raises(orc.OracleError, match="RankError"):
        orc.run_em(xs, 9, 3, seed=3)
    with pytest.raises(RankError):
        srm.fit(_subjects(srm, xs), srm.SrmConfig(k=9, iterations=3, seed=3), algorithm=algorithm)


def test_nccl_exchange_graph_bit_identical(srm, monkeypatch):
    """{NCCL all-gather of the E-step table, E-step, M-step} captured as one
    CUDA graph per rank (the N > 1 iteration, engine.capture_exchange) and
    replayed: on a one-rank NCCL group with the in-place all-gather forced
    into the graph (SRM_B200_FORCE_XGRAPH=1), the fit equals the
    single-rank native graph bit for bit, and the collective is issued from
    Python only twice (the eager first iteration and the capture)."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_1608_04647_b200.collectives import TorchCommunicator
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(4, 700, 150, 12, seed=17)
    cfg = srm.SrmConfig(k=12, iterations=6, seed=4)
    own = not dist.is_initialized()
    if own:
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    try:
        comm = TorchCommunicator()
        assert comm.device_collectives
        for algorithm in ("gram", "stream"):
            monkeypatch.setenv("SRM_B200_FORCE_XGRAPH", "1")
            before = comm.stats.allgather_calls
            a = srm.fit(_subjects(srm, xs), cfg, comm, algorithm=algorithm)
            assert comm.stats.allgather_calls - before == 2, algorithm
            monkeypatch.delenv("SRM_B200_FORCE_XGRAPH")
            b = srm.fit(_subjects(srm, xs), cfg, algorithm=algorithm)
            assert np.array_equal(a.S, b.S) and np.array_equal(a.sigma_s, b.sigma_s), algorithm
            assert np.array_equal(a.rho2, b.rho2) and a.log_likelihood == b.log_likelihood, algorithm
            for wa, wb in zip(a.W, b.W):
                assert np.array_equal(wa, wb), algorithm
    finally:
        if own:
            dist.destroy_process_group()


@pytest.mark.parametrize("k", [10, 64, 100])
def test_fp32_final_w_in_kernel_slicing_bit_identical(srm, monkeypatch, k):
    """fp32 X-hat: the final W_i = Xhat_i R_i with the A operand sliced from
    X-hat inside the kernel (kRowWX: fp32 tiles by TMA, int8 digits by slicer
    warps) equals the W formed from the stored int8 records (SRM_B200_OZW=
    records) bit for bit: same digits, same MMAs, same epilogue. Ragged V (a
    partial 128-voxel tile), one or two 64-feature halves, T = 260 (partial
    32-TR k-block)."""
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(4, 1500, 260, k, seed=37)
    xs = [x.astype(np.float32) for x in xs]
    xs[1] = xs[1][:1157]
    cfg = srm.SrmConfig(k=k, iterations=2, seed=3)
    out = []
    for mode in ("x", "records"):
        monkeypatch.setenv("SRM_B200_OZW", mode)
        eng = []
        out.append(srm.fit(_subjects(srm, xs), cfg, algorithm="gram", engine_out=eng))
        assert eng[0].gram_i8
    for wa, wb in zip(out[0].W, out[1].W):
        assert np.array_equal(wa, wb)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_final_w_feature_halves_on_one_cta_bit_identical(srm, monkeypatch, dtype):
    """K = 100 (two 64-feature halves): the final W with both halves of a
    128-voxel item on one persistent CTA (default; the second half's A operand
    is an L2 hit) equals the W with the halves on neighbouring CTAs
    (SRM_B200_OZW_ZSEQ=0) bit for bit -- the same tiles, a different CTA
    assignment. More items than CTAs (so CTAs loop), ragged V, partial k-block."""
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(4, 6000, 260, 100, seed=41)
    xs = [x.astype(dtype) for x in xs]
    xs[2] = xs[2][:5157]
    cfg = srm.SrmConfig(k=100, iterations=2, seed=5)
    out = []
    for mode in ("1", "0"):
        monkeypatch.setenv("SRM_B200_OZW_ZSEQ", mode)
        eng = []
        out.append(srm.fit(_subjects(srm, xs), cfg, algorithm="gram", engine_out=eng))
        assert eng[0].gram_i8
    for wa, wb in zip(out[0].W, out[1].W):
        assert np.array_equal(wa, wb)
