"""Diagnostic: Newton-Schulz iteration counts of the per-subject polar (SRM_R_SCAL[i][0])."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1608_04647_b200 import _lib, srm
from paper_1608_04647_b200.data import recipe_torch

n, V, T, K, iters = (int(a) for a in sys.argv[1:6])
xs, _, _ = recipe_torch(n, V, T, K, seed=0, dtype="f64")
subs = [srm.SubjectData(f"s{i}", x) for i, x in enumerate(xs)]
for it in (1, 2, 5, iters):
    out = []
    srm.fit(subs, srm.SrmConfig(k=K, iterations=it), engine_out=out, keep_on_device=True)
    eng = out[0]
    scal = eng.region(_lib.R_SCAL, torch.float64).reshape(-1, 8)[: eng.n_local, 0]
    print(f"after {it} iterations: NS steps per subject", scal.cpu().numpy().astype(int).tolist())
