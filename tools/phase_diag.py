"""Diagnostic: wall time of the host-side pieces of srm.fit's setup and collect phases."""
import functools
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1608_04647_b200 import engine, hostio, srm
from paper_1608_04647_b200.data import recipe_torch

acc = {}


def timed(owner, name, label=None):
    fn = getattr(owner, name)

    @functools.wraps(fn)
    def wrap(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        acc[label or name] = acc.get(label or name, 0.0) + time.perf_counter() - t0
        return r

    setattr(owner, name, wrap)


timed(engine.SrmEngine, "__init__", "engine_init")
timed(engine.SrmEngine, "close")
timed(hostio.PinnedRing, "get")
timed(hostio, "to_pinned")
timed(hostio, "to_host")
timed(srm, "rank_counts")
timed(srm, "_storage_for")
timed(srm, "gram_int8_bytes")
timed(srm, "choose_algorithm")
timed(torch.cuda, "mem_get_info")
timed(engine.SrmEngine, "small_results_to_host")
timed(engine.SrmEngine, "mu_host")
timed(engine.SrmEngine, "finalize_to_host")
timed(engine.SrmEngine, "start_mu_readback")
timed(srm, "ThreadPoolExecutor", "pool_create")
timed(srm.SrmConfig, "validate")
timed(srm, "_collect")

n, V, T, K, iters = (int(a) for a in sys.argv[1:6])
xs, _, _ = recipe_torch(n, V, T, K, seed=0, dtype="f64")
host = [x.cpu().pin_memory() for x in xs]
del xs
torch.cuda.empty_cache()
subs = [srm.SubjectData(f"s{i}", h) for i, h in enumerate(host)]
cfg = srm.SrmConfig(k=K, iterations=iters)
for rep in range(4):
    acc.clear()
    tm = {}
    t0 = time.perf_counter()
    m = srm.fit(subs, cfg, timings=tm)
    del m
    print(f"total {time.perf_counter() - t0:.4f}", {k: round(v * 1e3, 2) for k, v in tm.items()},
          {k: round(v * 1e3, 2) for k, v in acc.items()})
