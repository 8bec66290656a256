"""Numpy restatement of the int8 Gram's slice arithmetic (csrc/ozaki.cu) to
size the error of dropping the d-groups s + s' > dmax off the diagonal.

x = 2^e sum_s q_s 2^(-6-7s) (balanced base-128 digits below the column
maximum, 7 slices for fp64 X-hat, 4 for fp32); G ~= 2^(e_a+e_b) sum_d
2^(-12-7d) sum_{s+s'=d} Q_s^T Q_s'.  Prints, for the BASELINE recipe (one
cfg-2-sized subject), the normwise error of G, of B = S G / 2 and of
A^T A = B S^T / 4 against the fp64 product, with and without keeping every
d-group on the diagonal, and the orthonormality of W = X S^T M / 2 with M
from the approximate A^T A.  Host-only; a design probe, not a test.
"""

import sys
import os

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1608_04647_b200.data import recipe_numpy  # noqa: E402


def slices(x, nsl):
    e = np.frexp(np.abs(x).max(0))[1]
    y = x * np.ldexp(1.0, 6 - e)
    qs = []
    for _ in range(nsl):
        r = np.rint(y)
        qs.append(r)
        y = (y - r) * 128
    return qs, e


def gram(qs, e, dmax, keep_diag):
    nsl, T = len(qs), qs[0].shape[1]
    g = np.zeros((T, T))
    for d in range(0, min(2 * nsl - 2, 6) + 1):
        acc = np.zeros((T, T))
        for s in range(max(0, d - nsl + 1), min(d, nsl - 1) + 1):
            if d <= dmax:
                acc += qs[s].T @ qs[d - s]
            elif keep_diag:
                acc[np.diag_indices(T)] += (qs[s] * qs[d - s]).sum(0)
        g += acc * 2.0 ** (-12 - 7 * d)
    return g * np.ldexp(1.0, e[:, None] + e[None, :])


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def main():
    rng = np.random.default_rng(0)
    xs, _, _ = recipe_numpy(1, 30000, 1000, 50, seed=1)
    x = xs[0] - xs[0].mean(1, keepdims=True)
    for k in (50, 100):
        s = rng.standard_normal((k, 1000))
        for nsl in (7, 4):
            xx = x.astype(np.float32).astype(np.float64) if nsl == 4 else x
            gt = xx.T @ xx
            qs, e = slices(xx, nsl)
            a = xx @ s.T / 2
            for dmax, fix in ((6, False), (5, True), (4, True), (3, True), (3, False)):
                if nsl == 4 and dmax > 3 and dmax < 6:
                    continue
                g = gram(qs, e, dmax, fix)
                b, br = s @ g / 2, s @ gt / 2
                ata, atar = b @ s.T / 2, br @ s.T / 2
                w_, v = np.linalg.eigh(ata)
                w = a @ (v @ np.diag(w_ ** -0.5) @ v.T)
                print(f"K={k} nsl={nsl} dmax={dmax} diag={fix}: G {rel(g, gt):.2e} B {rel(b, br):.2e} "
                      f"AtA {rel(ata, atar):.2e} |W^T W - I| {np.abs(w.T @ w - np.eye(k)).max():.2e}")


if __name__ == "__main__":
    main()
