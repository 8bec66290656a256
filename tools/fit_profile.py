"""Diagnostic: host-side cProfile of one warm srm.fit (which Python calls hold the wall clock)."""
import cProfile
import pstats
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
for _ in range(2):
    m = srm.fit(subs, cfg)
    del m
pr = cProfile.Profile()
torch.cuda.synchronize()
t0 = time.perf_counter()
pr.enable()
m = srm.fit(subs, cfg)
torch.cuda.synchronize()
pr.disable()
print(f"fit {time.perf_counter() - t0:.4f} s")
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
