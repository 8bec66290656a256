"""The SRM subset of the reference's dense kernels on the device
(paper_1608_04647_b200.kernels -> srm_trace_ata / srm_add_diag /
srm_spd_inverse / srm_polar) against the golden vectors the real reference
produced (tests/golden/kernels.npz) and the reference's own test cases
(/root/reference/pkg/tests/test_kernels.py:52-163), restated here.
"""

import numpy as np
import pytest

from conftest import load_golden, nrel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kern():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_1608_04647_b200 import kernels

    return kernels


@pytest.fixture(scope="module")
def err():
    from paper_1608_04647_b200 import errors

    return errors


# ---------------------------------------------------------------- golden


def test_golden_spd_inverse(kern):
    g = load_golden("kernels")
    for i in range(5):
        out = kern.spd_inverse(g[f"spd_in{i}"])
        assert nrel(out, g[f"spd_out{i}"]) <= 1e-12, (i, nrel(out, g[f"spd_out{i}"]))
        assert np.array_equal(out, out.T)
    # cond 1e6 (test_kernels.py:119-126): within eps cond of the reference's own inverse
    out = kern.spd_inverse(g["spd_ill_in"])
    assert nrel(out, g["spd_ill_out"]) <= 1e-9
    assert np.max(np.abs(g["spd_ill_in"] @ out - np.eye(8))) <= 1e-8


def test_golden_spd_pivot(kern, err):
    g = load_golden("kernels")
    with pytest.raises(err.DefinitenessError) as ei:
        kern.spd_inverse(g["spd_bad_in"])
    assert ei.value.pivot == int(g["spd_bad_pivot"]) == 3


def test_golden_polar(kern):
    g = load_golden("kernels")
    for i in range(4):
        a = g[f"polar_in{i}"]
        w = kern.polar_orthogonal(a)
        ref = g[f"polar_out{i}"]
        assert nrel(w, ref) <= 1e-12, (i, nrel(w, ref))
        assert np.max(np.abs(w.T @ w - np.eye(a.shape[1]))) <= 1e-13


def test_golden_trace_ata(kern):
    g = load_golden("kernels")
    assert abs(kern.trace_ata(g["tata_in"]) - float(g["tata_out"])) <= 1e-13 * abs(float(g["tata_out"]))


# ------------------------------------------------ test_kernels.py restated


def test_trace_ata_cases(kern, err):
    assert kern.trace_ata(np.eye(2)) == 2.0
    assert kern.trace_ata(np.array([[1.0, 2.0], [3.0, 4.0]])) == 30.0
    rng = np.random.default_rng(2)
    a = rng.standard_normal((20, 6))
    assert abs(kern.trace_ata(a) - float(np.trace(a.T @ a))) <= 1e-10
    rng = np.random.default_rng(3)
    for _ in range(20):
        assert kern.trace_ata(rng.standard_normal((4, 3)) * rng.exponential()) >= 0.0
    assert kern.trace_ata(np.zeros((5, 4))) == 0.0
    assert kern.trace_ata(np.array([[1e-150]])) > 0.0
    with pytest.raises(err.InvalidInputError):
        kern.trace_ata(np.array([[1.0, np.inf]]))
    with pytest.raises(err.ShapeError):
        kern.trace_ata(np.zeros(3))


def test_add_diag_cases(kern, err):
    assert np.array_equal(kern.add_diag(np.zeros((3, 3)), 1.0), np.eye(3))
    assert np.array_equal(kern.add_diag(np.eye(2), -1.0), np.zeros((2, 2)))
    rng = np.random.default_rng(4)
    a = rng.standard_normal((8, 8))
    out = kern.add_diag(a, 0.5)
    off = ~np.eye(8, dtype=bool)
    assert np.array_equal(out[off], a[off])
    assert np.array_equal(np.diag(out), np.diag(a) + 0.5)
    with pytest.raises(err.ShapeError):
        kern.add_diag(np.zeros((2, 3)), 1.0)


def test_spd_inverse_cases(kern, err):
    assert np.allclose(kern.spd_inverse(np.eye(4)), np.eye(4))
    assert np.allclose(kern.spd_inverse(np.diag([2.0, 4.0])), np.diag([0.5, 0.25]))
    rng = np.random.default_rng(5)
    c = rng.standard_normal((6, 6))
    b = c.T @ c + np.eye(6)
    assert np.max(np.abs(b @ kern.spd_inverse(b) - np.eye(6))) <= 1e-10
    rng = np.random.default_rng(6)
    c = rng.standard_normal((5, 5))
    inv = kern.spd_inverse(c.T @ c + np.eye(5))
    assert np.array_equal(inv, inv.T)
    with pytest.raises(err.DefinitenessError) as ei:
        kern.spd_inverse(np.diag([1.0, -1.0, 2.0]))
    assert ei.value.pivot == 1
    rng = np.random.default_rng(7)
    vals = np.logspace(0, 6, 8)
    q = np.linalg.qr(rng.standard_normal((8, 8)))[0]
    a = q @ np.diag(vals) @ q.T
    a = 0.5 * (a + a.T)
    assert np.max(np.abs(a @ kern.spd_inverse(a) - np.eye(8))) <= 1e-8


def test_polar_cases(kern, err):
    rng = np.random.default_rng(8)
    q = np.linalg.qr(rng.standard_normal((7, 3)))[0]
    assert np.max(np.abs(kern.polar_orthogonal(q) - q)) <= 1e-12
    a = np.zeros((4, 2))
    a[0, 0], a[1, 1] = 2.0, 3.0
    expected = np.zeros((4, 2))
    expected[0, 0] = expected[1, 1] = 1.0
    assert np.max(np.abs(kern.polar_orthogonal(a) - expected)) <= 1e-12
    rng = np.random.default_rng(9)
    a = rng.standard_normal((30, 5))
    vals, vecs = np.linalg.eigh(a.T @ a)
    assert np.max(np.abs(kern.polar_orthogonal(a) - a @ (vecs @ np.diag(vals ** -0.5) @ vecs.T))) <= 1e-8
    rng = np.random.default_rng(10)
    for rows, cols in [(5, 5), (12, 3), (40, 7)]:
        w = kern.polar_orthogonal(rng.standard_normal((rows, cols)))
        assert np.max(np.abs(w.T @ w - np.eye(cols))) <= 1e-10
    with pytest.raises(err.RankError):
        kern.polar_orthogonal(np.ones((6, 2)))  # both columns identical
    with pytest.raises(err.ShapeError):
        kern.polar_orthogonal(np.ones((2, 4)))


# ------------------------------------------- conditioning (kernels.py:202-206)


def _conditioned(rows, cols, ratio, seed):
    rng = np.random.default_rng(seed)
    u = np.linalg.qr(rng.standard_normal((rows, cols)))[0]
    v = np.linalg.qr(rng.standard_normal((cols, cols)))[0]
    return u @ np.diag(np.logspace(0, np.log10(ratio), cols)) @ v.T, u @ v.T


@pytest.mark.parametrize("ratio", [1e-3, 1e-6, 1e-9, 1e-11])
def test_polar_ill_conditioned_resolved(kern, ratio):
    """sigma_min / sigma_max down to 1e-11 (the reference raises only below
    1e-12): W equals the exact polar factor to ~eps cond(A) -- the Gram route
    A (A^T A)^{-1/2} loses ~eps cond(A)^2 -- and is orthonormal to roundoff."""
    for rows, cols, seed in [(300, 12, 1), (4000, 40, 2), (50, 50, 3)]:
        a, exact = _conditioned(rows, cols, ratio, seed)
        w = kern.polar_orthogonal(a)
        assert nrel(w, exact) <= max(1e-13, 50 * 2.2e-16 / ratio), (rows, cols, ratio, nrel(w, exact))
        assert np.max(np.abs(w.T @ w - np.eye(cols))) <= 1e-13


@pytest.mark.parametrize("ratio", [1e-13, 1e-15, 0.0])
def test_polar_rank_deficient_rejected(kern, err, ratio):
    a, _ = _conditioned(500, 10, max(ratio, 1e-300), 4)
    if ratio == 0.0:
        a[:, 3] = a[:, 7]
    with pytest.raises(err.RankError):
        kern.polar_orthogonal(a)


def test_polar_large_tall(kern):
    """V = 200,000 x K = 100 (cfg 3's A_i): four TSQR levels."""
    rng = np.random.default_rng(11)
    a = rng.standard_normal((200000, 100))
    w = kern.polar_orthogonal(a)
    u, _, vt = np.linalg.svd(a, full_matrices=False)
    assert nrel(w, u @ vt) <= 1e-12
    assert np.max(np.abs(w.T @ w - np.eye(100))) <= 1e-13


def test_step_api_rank_error_matches_reference(kern, err):
    """srm.m_step_subject on an S with two equal rows: A = Xhat S^T / 2 has two
    equal columns, the reference's gesdd polar raises RankError."""
    from paper_1608_04647_b200 import srm

    rng = np.random.default_rng(12)
    s = rng.standard_normal((3, 40))
    s[2] = s[0]
    with pytest.raises(err.RankError):
        srm.m_step_subject(rng.standard_normal((200, 40)), s, 1.0)
