"""Kernel timeline of one bench step from CUPTI (torch.profiler): every kernel
of a complete fit -- the one-time Gram, the init, the EM iterations as graph
replays, the final W -- with its real start / end on the device (no
serialisation, unlike ncu), so the per-iteration critical path, the overlap of
the side lanes and the gaps between kernels are visible.

    python tools/chain_probe.py --config cfg2 [--out gpurun_out/chain_cfg2.json]

Prints per phase: the span, the busy time of each kernel and the idle gaps;
for the iterations, one iteration's kernel sequence with start offsets.
With --eager one extra iteration runs eagerly between cudaProfilerStart/Stop
(for ``ncu --profile-from-start off``)."""
import argparse
import json
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1608_04647_b200.data import config_by_name, recipe_torch  # noqa: E402
from paper_1608_04647_b200.engine import SrmEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--subjects", type=int, default=None)
ap.add_argument("--out", default=None)
ap.add_argument("--eager", action="store_true")
args = ap.parse_args()
cfg = config_by_name(args.config)
n = args.subjects or cfg["n_subjects"]
V, T, K, it = cfg["n_voxels"], cfg["n_trs"], cfg["k"], cfg["iterations"]
xs, _, _ = recipe_torch(n, V, T, K, seed=0, smooth=cfg["smooth"], dtype=cfg["dtype"])
eng = SrmEngine([V] * n, T, K, it, storage=cfg["dtype"], gram=True, gram_i8=True)
eng.load(xs)
del xs
torch.cuda.empty_cache()
eng.prepare_gram()
eng.init_mapping(0, 0)
draws = eng.amat.clone()


def step(marks=None):
    def mark(name):
        if marks is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append((name, e))

    mark("start")
    eng.reset()
    eng.amat.copy_(draws)
    eng.prepare_gram()
    mark("gram")
    eng.init_kernels()
    mark("init")
    for i in range(it):
        if eng._graph is not None:
            eng.replay()
        else:
            eng.step()
            eng.capture()
        mark(f"it{i}")
    eng.finalize()
    mark("finalize")


for _ in range(2):
    step()
torch.cuda.synchronize()
if args.eager:  # under ncu: no CUPTI timeline, one eager iteration between profiler start / stop
    torch.cuda.profiler.start()
    eng.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    eng.raise_status()
    sys.exit(0)
marks = []
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    step(marks)
    torch.cuda.synchronize()
eng.raise_status()
spans = [(marks[j + 1][0], marks[j][1].elapsed_time(marks[j + 1][1])) for j in range(len(marks) - 1)]

kern = []
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA and ev.time_range.elapsed_us() > 0:
        nm = ev.name
        if "memcpy" in nm.lower() or "memset" in nm.lower():
            kind = "copy"
        else:
            kind = "kernel"
        kern.append({"name": nm, "start": ev.time_range.start, "end": ev.time_range.end, "kind": kind})
kern.sort(key=lambda k: k["start"])
t0 = kern[0]["start"]


def short(nm):
    nm = nm.replace("void ", "").replace("srm::", "").replace("(anonymous namespace)::", "")
    return nm.split("(")[0][:40]


# phases by the event spans, in device time from the first kernel
bounds = []
acc = 0.0
for name, ms in spans:
    bounds.append((name, acc * 1e3, (acc + ms) * 1e3))
    acc += ms
out = {"config": args.config, "subjects": n, "spans_ms": dict(spans), "phases": {}}
# assign kernels to phases by cumulative position (kernel starts relative to the first)
for name, lo, hi in bounds:
    ks = [k for k in kern if lo <= k["start"] - t0 < hi]
    if not ks:
        continue
    busy = defaultdict(float)
    for k in ks:
        busy[short(k["name"])] += k["end"] - k["start"]
    # union of kernel intervals -> idle gaps inside the phase
    iv = sorted((k["start"], k["end"]) for k in ks)
    union, cur = 0.0, list(iv[0])
    for s, e in iv[1:]:
        if s > cur[1]:
            union += cur[1] - cur[0]
            cur = [s, e]
        else:
            cur[1] = max(cur[1], e)
    union += cur[1] - cur[0]
    span = ks[-1]["end"] - ks[0]["start"]
    out["phases"][name] = {"span_us": span, "busy_union_us": union, "idle_us": span - union,
                           "kernels_us": dict(sorted(busy.items(), key=lambda x: -x[1]))}
    if name == "gram":
        out["gram_timeline"] = [(short(k["name"]), round(k["start"] - ks[0]["start"], 1),
                                 round(k["end"] - k["start"], 1)) for k in ks]
    if name == "it1":
        out["iteration_timeline"] = [(short(k["name"]), round(k["start"] - ks[0]["start"], 1),
                                      round(k["end"] - k["start"], 1)) for k in ks]
print(json.dumps({"config": out["config"], "spans_ms": out["spans_ms"]}, indent=None))
for name, ph in out["phases"].items():
    if name.startswith("it") and name not in ("it0", "it1"):
        continue
    print(f"== {name}: span {ph['span_us']:.1f} us, busy {ph['busy_union_us']:.1f}, idle {ph['idle_us']:.1f}")
    for k, v in list(ph["kernels_us"].items())[:14]:
        print(f"   {k:42s} {v:9.1f} us")
print("== iteration 1 timeline (name, start us, duration us)")
for row in out.get("iteration_timeline", []):
    print("  ", row)
if args.out:
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
