"""Where one bench step goes: CUDA events around each phase of a complete fit
(reset + draw restore, the one-time Gram, the device init, the EM iterations as
graph replays, the final W) on a BASELINE config, averaged over a few steps."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_04647_b200 import srm  # noqa: E402
from paper_1608_04647_b200.data import config_by_name, recipe_torch  # noqa: E402
from paper_1608_04647_b200.engine import SrmEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--steps", type=int, default=5)
args = ap.parse_args()
cfg = config_by_name(args.config)
V, T, K, it = cfg["n_voxels"], cfg["n_trs"], cfg["k"], cfg["iterations"]
xs, _, _ = recipe_torch(cfg["n_subjects"], V, T, K, seed=0, smooth=cfg["smooth"], dtype=cfg["dtype"])
eng = SrmEngine([V] * cfg["n_subjects"], T, K, it, storage=cfg["dtype"], gram=True, gram_i8=True)
eng.load(xs)
del xs
torch.cuda.empty_cache()
eng.prepare_gram()
eng.init_mapping(0, 0)
draws = eng.amat.clone()
names = ["reset", "gram", "init", "iterations", "finalize"]
acc = {n: 0.0 for n in names}
for s in range(args.steps + 1):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
    ev[0].record()
    eng.reset()
    eng.amat.copy_(draws)
    ev[1].record()
    eng.prepare_gram()
    ev[2].record()
    eng.init_kernels()
    ev[3].record()
    for i in range(it):
        if eng._graph is not None:
            eng.replay()
        else:
            eng.step()
            eng.capture()
    ev[4].record()
    eng.finalize()
    ev[5].record()
    torch.cuda.synchronize()
    if s > 0:
        for j, n in enumerate(names):
            acc[n] += ev[j].elapsed_time(ev[j + 1]) / args.steps
eng.raise_status()
tot = sum(acc.values())
print(args.config, " ".join(f"{n} {v:.3f} ms" for n, v in acc.items()), f"total {tot:.3f} ms",
      f"per iteration {acc['iterations'] / it:.4f} ms")
