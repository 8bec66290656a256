"""Per-iteration error of each fp32 device path against the oracle on a
cfg3-shaped slice (V = 200,000 / T = 2,000 / K = 100 scaled down by --scale),
plus cond(A_i) of the oracle's M-steps: which stage sets the fp32 error."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import srm_oracle as orc  # noqa: E402
from paper_1608_04647_b200 import srm  # noqa: E402
from paper_1608_04647_b200.data import recipe_torch  # noqa: E402


def nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4)
ap.add_argument("--v", type=int, default=50000)
ap.add_argument("--t", type=int, default=2000)
ap.add_argument("--k", type=int, default=100)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--nsub", type=int, default=16, help="recipe's subject count (seeds)")
args = ap.parse_args()
xs = [recipe_torch(args.nsub, args.v, args.t, args.k, seed=0, dtype="f32", first_subject=i, count=1)[0][0]
      .cpu().numpy() for i in range(args.n)]
ref = list(orc.em_iterations(xs, args.k, args.iters, seed=0, workers=16))
xh = [orc.center_rows(x)[0] for x in xs]
print("cond(A_0) per iteration:", ["%.2f" % np.linalg.cond(0.5 * (xh[0] @ r["S"].T)) for r in ref], flush=True)
variants = {
    "tc_stream": dict(algorithm="stream", tensor_cores=True),
    "gram_i8": dict(algorithm="gram"),
    "gram_f64": dict(algorithm="gram", gram_int8=False),
    "stream_f64": dict(algorithm="stream", tensor_cores=False),
    "exact": dict(exact_polar=True),
}
for name, kw in variants.items():
    rows = []

    def cb(st):
        r = ref[st.iteration]
        rows.append((nrel(st.S, r["S"]), nrel(st.sigma_s, r["sigma_s"]), nrel(st.rho2, r["rho2"]),
                     max(nrel(w, rw) for w, rw in zip(st.W, r["W"]))))

    eng = []
    srm.fit([srm.SubjectData(f"s{j}", x) for j, x in enumerate(xs)], srm.SrmConfig(k=args.k, iterations=args.iters),
            on_iteration=cb, engine_out=eng, **kw)
    e = eng[-1]
    print(f"{name:10s} gram={e.gram} i8={e.gram_i8} tc={e.tc} exact={e.exact_polar}", flush=True)
    for i, r in enumerate(rows):
        print(f"   it{i}: S {r[0]:.2e} sigma {r[1]:.2e} rho2 {r[2]:.2e} W {r[3]:.2e}", flush=True)
