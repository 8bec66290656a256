"""Diagnostic: Jacobi sweeps per subject and eig_polar time on a cfg2-shaped plan."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1608_04647_b200 import _lib
from paper_1608_04647_b200.data import recipe_torch
from paper_1608_04647_b200.engine import SrmEngine

n, V, T, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
xs, _, _ = recipe_torch(n, V, T, K, seed=0, dtype="f64")
eng = SrmEngine([V] * n, T, K, 30, storage="f64")
eng.load(xs)
eng.init_mapping(0, 0)
scal = eng.region(_lib.R_SCAL).view(n, 8)
for it in range(12):
    prof = dict(eng.profile_iteration())
    print(it, "iters", scal[:, 0].tolist()[:6], {k: round(v, 3) for k, v in prof.items()})
