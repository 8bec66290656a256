"""One line per bench JSON file: the headline numbers, CPU sweep and kernel split."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    if d.get("impl") == "reference":
        print(f, "REFERENCE value %.3e ms/step %.0f" % (d["value"], d["ms_per_step"]), d["cpu_baseline"]["sample"])
        continue
    r, e, c = d["roofline"], d.get("e2e") or {}, d.get("cpu_baseline") or {}
    print(f"{f}: {d['config']['workload'][:60]} algo={d['algorithm']} ms/step {d['ms_per_step']:.2f} "
          f"value {d['value']:.3e} e2e {e.get('value', 0):.3e} ({e.get('seconds_per_fit', 0):.3f} s) "
          f"roofline {r['kernel']} {r['frac']:.2f} cpu {c.get('value', 0):.2e} launches {d['gpu_launches']} "
          f"clocks {d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}")
    print("   hbm:", {k: round(v["frac"], 2) for k, v in d["roofline_hbm"]["kernels"].items()},
          "streaming-equivalent %.2f" % d["roofline_hbm"]["streaming_equivalent"]["frac"])
    print("   per-iteration ms:", {k: round(v, 3) for k, v in d["kernel_ms"]["per_iteration_ms"].items()})
    print("   one-time ms:", {k: round(v, 2) for k, v in d["kernel_ms"]["one_time_ms"].items()})
    if c.get("sweep"):
        print("   cpu sweep:", {k: "%.2e" % v for k, v in c["sweep"].items()}, c.get("blas"), c.get("cpu"))
