"""Diagnostic: int8-sliced Gram vs the fp64 DMMA Gram (accuracy and time).

usage: python tools/oz_check.py n V T [heavy]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1608_04647_b200 import _lib
from paper_1608_04647_b200.data import recipe_torch
from paper_1608_04647_b200.engine import SrmEngine

n, V, T = (int(a) for a in sys.argv[1:4])
heavy = len(sys.argv) > 4
xs, _, _ = recipe_torch(n, V, T, 10, seed=3)
if heavy:  # heavy-tailed columns: a few large spikes
    g = torch.Generator(device="cuda").manual_seed(5)
    for x in xs:
        idx = torch.randint(0, x.numel(), (max(1, x.numel() // 10000),), device=x.device, generator=g)
        x.view(-1)[idx] *= 50.0
ragged = [V - 37 * j for j in range(n)]
xs = [x[:v] for x, v in zip(xs, ragged)]
res = {}
for i8 in (False, True):
    eng = SrmEngine(ragged, T, 10, 2, gram=True, gram_i8=i8)
    assert eng.gram_i8 == i8, "flag not effective"
    eng.load(xs)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.prepare_gram()
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
    eng.raise_status()
    G = eng.region(_lib.R_GRAM, torch.float64).view(n, eng.ldx, eng.ldx).clone()
    res[i8] = (G, ms)
    print(f"i8={i8}: prepare_gram {ms:.3f} ms")
    del eng
    torch.cuda.empty_cache()
G0, G1 = res[False][0], res[True][0]
d = (G1 - G0)
rel = (d.norm() / G0.norm()).item()
maxrel = (d.abs().amax() / G0.abs().amax()).item()
diag = torch.diagonal(G0, dim1=1, dim2=2)
scale = torch.sqrt(diag.unsqueeze(2) * diag.unsqueeze(1)).clamp_min(1e-300)
entry = (d.abs() / scale).amax().item()
sym = (G1 - G1.transpose(1, 2)).abs().max().item()
print(f"normwise rel {rel:.3e}  max|d|/max|G| {maxrel:.3e}  max |d_ab|/sqrt(G_aa G_bb) {entry:.3e}  asym {sym:.1e}")
print(f"speedup {res[False][1] / res[True][1]:.2f}x")
