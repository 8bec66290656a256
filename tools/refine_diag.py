"""Which polar stage raises the conditioning warning on an fp32 K = 100 fit:
reads status[3] and the per-subject refine flags (scal[i][1]) after the init
and after every iteration (one subject window at a time)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_04647_b200 import _lib  # noqa: E402
from paper_1608_04647_b200.data import recipe_numpy  # noqa: E402
from paper_1608_04647_b200.engine import SrmEngine  # noqa: E402

for case in ("ragged330", "smooth260"):
    if case == "ragged330":
        xs, _, _ = recipe_numpy(3, 2600, 330, 100, seed=23, dtype="f32")
        xs = [x[: 2600 - 97 * i] for i, x in enumerate(xs)]
    else:
        xs, _, _ = recipe_numpy(3, 1500, 260, 100, seed=4, dtype="f32")
    T = xs[0].shape[1]
    eng = SrmEngine([x.shape[0] for x in xs], T, 100, 4, storage="f32", gram=True, gram_i8=True)
    eng.load(xs)
    eng.prepare_gram()
    eng.init_mapping(4, 0)
    torch.cuda.synchronize()
    scal = eng.region(_lib.R_SCAL).view(eng.n_local, 8)
    print(case, "init: warn", eng.status()[3], "ns iters", scal[:, 0].tolist(), "refine ok", scal[:, 1].tolist(), "steps", scal[:, 2].tolist())
    for it in range(4):
        eng.step()
        torch.cuda.synchronize()
        print(case, f"it{it}: warn", eng.status()[3], "ns iters", scal[:, 0].tolist(), "refine ok", scal[:, 1].tolist(), "steps", scal[:, 2].tolist())
    eng.close()
