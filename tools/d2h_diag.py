"""Diagnostic: D2H strategies for the 480 MB W read-back, and fit-to-fit variance."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

x = torch.randn(1_200_000, 50, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for name in ["cpu", "np_empty", "pinned", "np_empty_prefault"]:
    for rep in range(3):
        t0 = time.perf_counter()
        if name == "cpu":
            h = x.cpu().numpy()
        elif name == "np_empty":
            h = np.empty((1_200_000, 50))
            torch.from_numpy(h).copy_(x)
        elif name == "pinned":
            ht = torch.empty((1_200_000, 50), dtype=torch.float64, pin_memory=True)
            ht.copy_(x)
            h = ht.numpy()
        else:
            h = np.empty((1_200_000, 50))
            h.fill(0)
            t1 = time.perf_counter()
            torch.from_numpy(h).copy_(x)
        torch.cuda.synchronize()
        print(name, rep, "%.4f" % (time.perf_counter() - t0))
        del h
