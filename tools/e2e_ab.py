"""Diagnostic: e2e phases of srm.fit with and without init_overlap, interleaved."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1608_04647_b200 import srm
from paper_1608_04647_b200.data import recipe_torch

n, V, T, K, iters = (int(a) for a in sys.argv[1:6])
xs, _, _ = recipe_torch(n, V, T, K, seed=0, dtype="f64")
host = [x.cpu().pin_memory() for x in xs]
del xs
torch.cuda.empty_cache()
subs = [srm.SubjectData(f"s{i}", h) for i, h in enumerate(host)]
cfg = srm.SrmConfig(k=K, iterations=iters)
srm.fit(subs, cfg)
for rep in range(5):
    for ov in (True, False):
        tm = {}
        t0 = time.perf_counter()
        srm.fit(subs, cfg, timings=tm, init_overlap=ov)
        print(f"overlap={ov} total {time.perf_counter() - t0:.3f}", {k: round(v, 4) for k, v in tm.items()})
