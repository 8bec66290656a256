"""Diagnostic: which part of the pipelined load bounds it (cfg2 shape)."""
import sys, time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1608_04647_b200 import hostio
from paper_1608_04647_b200.data import recipe_torch
from paper_1608_04647_b200.engine import SrmEngine

n, V, T, K = 40, 30000, 1000, 50
xs, _, _ = recipe_torch(n, V, T, K, seed=0, dtype="f64")
host = [x.cpu().pin_memory() for x in xs]
del xs
torch.cuda.empty_cache()
eng = SrmEngine([V] * n, T, K, 20, storage="f64", gram=True, gram_i8=True)
def run(gaussians, gram, label):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    eng.load(host, gaussians=gaussians, gram=gram)
    torch.cuda.synchronize(); print(label, "%.4f" % (time.perf_counter() - t0))
run(None, False, "upload+demean")
run(None, True, "upload+demean+gram")
pool = ThreadPoolExecutor(16)
t0 = time.perf_counter()
arrs = list(pool.map(lambda j: np.random.default_rng((0, j)).standard_normal((V, K)), range(n)))
print("draws 16 threads %.4f" % (time.perf_counter() - t0))
run(list(arrs), True, "upload+demean+gram+g0(arrays)")
ring = hostio.PinnedRing.get(eng.device, V * K * 8, nslots=16, n_items=n)
def draw(j):
    ring.wait_free(j)
    np.random.default_rng((0, j)).standard_normal(out=ring.view(j, (V, K)))
    return (ring, j)
t0 = time.perf_counter()
futs = [pool.submit(draw, j) for j in range(n)]
run(futs, True, "upload+demean+gram+g0(ring)")
