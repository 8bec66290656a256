"""Subject containers and the BASELINE.json synthetic generative recipe.

``SubjectData`` mirrors ``factorfit.data_io.SubjectData``
(``/root/reference/pkg/src/factorfit/data_io.py:81-95``).

The generators implement the recipe every BASELINE config names (the
paper's fMRI datasets are not available; seeded synthetic data of the same
shapes stands in for them):

    S ~ N(0,1)^{K x T};  W_i = Q of QR(N(0,1)^{V x K}) (cfg 4: each column
    first smoothed along the voxel axis by a Gaussian, sigma = 5 voxels);
    rho_i ~ U[0.5, 1.5];  X_i = W_i S + E_i, E_i ~ N(0, rho_i^2);
    each X_i row-centred, then cast to the config dtype.

Two pinned RNG stream layouts:

* ``recipe_numpy`` (host): S from ``default_rng([seed, 0])``, subject i from
  ``default_rng([seed, 1, i])`` drawing G (V x K), rho, then E (V x T).
* ``recipe_torch`` (device, counter-based Philox): S from a CUDA generator
  seeded ``seed * 1_000_003``, subject i from one seeded
  ``seed * 1_000_003 + 1 + i``.  The CPU oracle consumes the same bytes by
  copying the generated tensors to the host.
"""

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Optional

import numpy as np

__all__ = ["SubjectData", "recipe_numpy", "recipe_torch", "CONFIGS", "config_by_name"]


@dataclass
class SubjectData:
    """One subject's voxels-by-TRs matrix plus optional voxel coordinates."""

    subject_id: str
    X: object
    grid: Optional[object] = None

    @property
    def n_voxels(self):
        return self.X.shape[0]

    @property
    def n_trs(self):
        return self.X.shape[1]


# BASELINE.json "configs" (subjects, voxels, TRs, k, dtype, iterations, smooth)
CONFIGS = {
    "cfg1": dict(n_subjects=10, n_voxels=5000, n_trs=500, k=50, dtype="f64", iterations=10, smooth=None),
    "cfg2": dict(n_subjects=40, n_voxels=30000, n_trs=1000, k=50, dtype="f64", iterations=20, smooth=None),
    "cfg3": dict(n_subjects=16, n_voxels=200000, n_trs=2000, k=100, dtype="f32", iterations=10, smooth=None),
    "cfg4": dict(n_subjects=256, n_voxels=50000, n_trs=1000, k=64, dtype="f32", iterations=10, smooth=5.0),
    "cfg5": dict(n_subjects=128, n_voxels=100000, n_trs=1000, k=100, dtype="f32", iterations=5, smooth=None),
}


def config_by_name(name):
    return dict(CONFIGS[name])


def _gauss_kernel(sigma):
    radius = int(4.0 * sigma + 0.5)
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    w = np.exp(-0.5 * (x / sigma) ** 2)
    return w / w.sum()


def _smooth_np(g, sigma):
    w = _gauss_kernel(sigma)
    out = np.empty_like(g)
    for j in range(g.shape[1]):
        out[:, j] = np.convolve(g[:, j], w, mode="same")
    return out


def _subject_np(seed, i, n_voxels, n_trs, k, shared, smooth, dtype):
    rng = np.random.default_rng([seed, 1, i])
    g = rng.standard_normal((n_voxels, k))
    if smooth:
        g = _smooth_np(g, smooth)
    q, _ = np.linalg.qr(g)
    rho = rng.uniform(0.5, 1.5)
    x = q @ shared
    x += rho * rng.standard_normal((n_voxels, n_trs))
    x -= x.mean(axis=1, keepdims=True)
    return x.astype(dtype, copy=False), rho


def recipe_numpy(n_subjects, n_voxels, n_trs, k, seed=0, smooth=None, dtype="f64",
                 first_subject=0, count=None, threads=8):
    """Host generator; returns (list of X_i, S, rho list) for subjects
    ``first_subject .. first_subject + count``."""
    np_dt = np.float64 if dtype == "f64" else np.float32
    shared = np.random.default_rng([seed, 0]).standard_normal((k, n_trs))
    count = n_subjects - first_subject if count is None else count
    idx = list(range(first_subject, first_subject + count))
    with ThreadPoolExecutor(max(1, min(threads, len(idx)))) as pool:
        out = list(pool.map(lambda i: _subject_np(seed, i, n_voxels, n_trs, k, shared, smooth, np_dt), idx))
    return [o[0] for o in out], shared, [o[1] for o in out]


def recipe_torch(n_subjects, n_voxels, n_trs, k, seed=0, smooth=None, dtype="f32",
                 first_subject=0, count=None, device="cuda"):
    """Device generator (Philox); returns (list of CUDA X_i, S, rho list)."""
    import torch

    t_dt = torch.float64 if dtype == "f64" else torch.float32
    gen = torch.Generator(device=device)
    gen.manual_seed(seed * 1_000_003)
    shared = torch.randn((k, n_trs), generator=gen, device=device, dtype=torch.float64)
    count = n_subjects - first_subject if count is None else count
    xs, rhos = [], []
    if smooth:
        w = torch.from_numpy(_gauss_kernel(smooth)).to(device).view(1, 1, -1)
    for i in range(first_subject, first_subject + count):
        gen.manual_seed(seed * 1_000_003 + 1 + i)
        g = torch.randn((n_voxels, k), generator=gen, device=device, dtype=torch.float64)
        if smooth:
            g = torch.nn.functional.conv1d(g.t().unsqueeze(1), w, padding=w.shape[-1] // 2)
            g = g.squeeze(1).t().contiguous()
        q, _ = torch.linalg.qr(g)
        rho = float(torch.rand((1,), generator=gen, device=device, dtype=torch.float64).item()) + 0.5
        x = torch.randn((n_voxels, n_trs), generator=gen, device=device, dtype=t_dt)
        x.mul_(rho)
        x.add_((q @ shared).to(t_dt))
        x.sub_(x.mean(dim=1, keepdim=True))
        del g, q
        xs.append(x)
        rhos.append(rho)
    return xs, shared, rhos
