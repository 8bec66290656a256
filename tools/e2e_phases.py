"""Per-phase wall seconds of srm.fit on pinned host arrays (the bench's e2e
leg), from fit's synchronising `timings` clock, beside the unsynchronised
total.  usage: python tools/e2e_phases.py [cfg2]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1608_04647_b200 import srm  # noqa: E402
from paper_1608_04647_b200.data_io import SubjectData  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
from paper_1608_04647_b200.data import config_by_name  # noqa: E402

cfg = config_by_name(name)
n, V, T, K = cfg["n_subjects"], cfg["n_voxels"], cfg["n_trs"], cfg["k"]
dt = np.float64 if cfg["dtype"] == "f64" else np.float32
rng = np.random.default_rng(0)
host = []
for j in range(n):
    t = torch.empty((V, T), dtype=torch.float64 if dt == np.float64 else torch.float32).pin_memory()
    t.normal_()
    host.append(t)
subjects = [SubjectData(f"sub-{j:04d}", host[j]) for j in range(n)]
conf = srm.SrmConfig(k=K, iterations=cfg["iterations"], seed=0)
srm.fit(subjects, conf)
out = {}
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    srm.fit(subjects, conf)
    torch.cuda.synchronize()
    out.setdefault("total_s", []).append(time.perf_counter() - t0)
tm = {}
torch.cuda.synchronize()
t0 = time.perf_counter()
srm.fit(subjects, conf, timings=tm)
torch.cuda.synchronize()
out["total_with_phase_syncs_s"] = time.perf_counter() - t0
out["phases_s"] = tm
print(json.dumps(out))
