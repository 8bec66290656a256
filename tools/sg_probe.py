"""Per-iteration stage times on cfg 2 (40 x 30000 x 1000, K = 50, fp64, int8
Gram path), eager with events between kernels, median of five iterations;
with SRM_B200_SG_PER_TILE=1 in the environment B = S G / 2 runs per tile.

    python tools/sg_probe.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_04647_b200.data import recipe_torch  # noqa: E402
from paper_1608_04647_b200.engine import SrmEngine  # noqa: E402

V, T, K, N = 30000, 1000, 50, 40
xs, _, _ = recipe_torch(N, V, T, K, seed=0, dtype="f64")
eng = SrmEngine([V] * N, T, K, 40, storage="f64", gram=True, gram_i8=True, device=torch.device("cuda:0"))
eng.load(xs)
eng.init_mapping(0, 0)
eng.prepare_gram()
eng.step(None)
torch.cuda.synchronize()
ts = {}
for _ in range(6):
    seen = {}
    for name, t in eng.profile_iteration():
        seen[name] = seen.get(name, 0) + 1
        ts.setdefault(name if seen[name] == 1 else f"{name}#{seen[name]}", []).append(t)
fin = {}
for _ in range(2):
    for name, t in eng.profile_finalize():
        fin.setdefault(name, []).append(t)
print(json.dumps({"per_iteration_ms": {k: float(np.median(v[1:])) for k, v in ts.items()},
                  "finalize_ms": {k: float(np.median(v)) for k, v in fin.items()}}), flush=True)


# phases of a timed fit (events on the engine stream): Gram precompute, 20
# replayed iterations, final W
eng.reset()
eng.init_mapping(0, 0)
st = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
torch.cuda.synchronize()
ev[0].record(st)
eng.prepare_gram()
ev[1].record(st)
for it in range(20):
    if eng._graph is not None:
        eng.replay()
    else:
        eng.step(None)
        eng.capture()
ev[2].record(st)
eng.finalize()
ev[3].record(st)
torch.cuda.synchronize()
print(json.dumps({"phase_ms": {"prepare_gram": ev[0].elapsed_time(ev[1]), "iterations_20": ev[1].elapsed_time(ev[2]),
                               "finalize": ev[2].elapsed_time(ev[3])}}), flush=True)

# Newton-Schulz steps of the last polar per subject (SRM_R_SCAL[i][0])
SRM_R_SCAL = 12  # include/srm_b200.h
scal = eng.region(SRM_R_SCAL, torch.float64)
print(json.dumps({"ns_steps": scal.view(-1, 8)[:, 0].cpu().tolist()}), flush=True)
