"""Diagnostic: per-phase wall time of srm.fit on pinned host arrays (cfg shape from argv)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1608_04647_b200 import srm
from paper_1608_04647_b200.data import recipe_torch

n, V, T, K, iters = (int(a) for a in sys.argv[1:6])
dt = sys.argv[6] if len(sys.argv) > 6 else "f64"
xs, _, _ = recipe_torch(n, V, T, K, seed=0, dtype=dt)
host = [x.cpu().pin_memory() for x in xs]
del xs
torch.cuda.empty_cache()
subs = [srm.SubjectData(f"s{i}", h) for i, h in enumerate(host)]
cfg = srm.SrmConfig(k=K, iterations=iters)
srm.fit(subs, cfg)
for _ in range(2):
    tm = {}
    t0 = time.perf_counter()
    srm.fit(subs, cfg, timings=tm)
    print("total %.3f" % (time.perf_counter() - t0), {k: round(v, 4) for k, v in tm.items()})
t0 = time.perf_counter(); srm.fit(subs, cfg); print("untimed total %.3f" % (time.perf_counter() - t0))
# numpy (pageable) inputs, the reference API's usual case
nps = [srm.SubjectData(f"s{i}", h.numpy()) for i, h in enumerate(host)]
for _ in range(2):
    tm = {}
    t0 = time.perf_counter()
    srm.fit(nps, cfg, timings=tm)
    print("numpy total %.3f" % (time.perf_counter() - t0), {k: round(v, 4) for k, v in tm.items()})
