"""Small driver for ncu captures of the one-time Gram stages: load n subjects
of a config's shape (fp32 or fp64), run srm_prepare_gram twice (the second is
the one to profile: ncu -s <kernels of the first> ...)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_04647_b200.data import config_by_name, recipe_torch  # noqa: E402
from paper_1608_04647_b200.engine import SrmEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--subjects", type=int, default=16)
ap.add_argument("--finalize", action="store_true")
args = ap.parse_args()
cfg = config_by_name(args.config)
xs, _, _ = recipe_torch(cfg["n_subjects"], cfg["n_voxels"], cfg["n_trs"], cfg["k"], seed=0, dtype=cfg["dtype"],
                        count=args.subjects)
eng = SrmEngine([cfg["n_voxels"]] * args.subjects, cfg["n_trs"], cfg["k"], 2, storage=cfg["dtype"], gram=True,
                gram_i8=True)
eng.load(xs)
del xs
for _ in range(2):
    eng.prepare_gram()
    torch.cuda.synchronize()
if args.finalize:
    eng.init_mapping(0, 0)
    for _ in range(2):
        eng.step()
    for _ in range(2):
        eng.finalize()
torch.cuda.synchronize()
eng.raise_status()
print("ok", eng.profile_gram())
