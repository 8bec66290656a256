#!/usr/bin/env python
"""Benchmark of the SRM EM fit on B200 (BASELINE.json metric and config).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
    python bench.py --impl reference ...      # the reference CPU arithmetic

A *step* is one EM iteration over every subject of the workload (srm.py:254-287:
E-step reduction, K x K tail, M-step over all subjects).  ``value`` is the
whole-job subject*voxel*TR/s per iteration with X already resident in HBM,
timed with CUDA events over a K-step fit (max over ranks): the one-time Gram
precompute (when that path is chosen) and the final W are inside the timed
region, demean and the reference initialisation are not; ``e2e`` is the
same metric through the public API ``srm.fit`` on pinned host arrays, host to
device copies, the reference initialisation and the read-back of the model
included.  The default workload is BASELINE config 2 (40 subjects x 30,000
voxels x 1,000 TRs, k=50, fp64); subjects are sharded across ranks (strong
scaling, cli.py:82-85 contiguous shards).

Under torchrun (N > 1) every rank drives one GPU over NCCL; the per-iteration
exchange is one all-gather of the ordered E-step table.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SRM EM subject·voxel·TR/s per iteration; achieved HBM GB/s vs B200 peak"
UNIT = "subject·voxel·TR/s"
DMMA_PEAK_TFLOPS = 37.1  # tools/fp64_peak.cu on this pool's B200 (mma.sync m8n8k4 f64)
FALLBACK_HBM_GBS = 6650.0
TF32_PEAK_TFLOPS = 1664.3 / 2  # tf32 MMA rate = half of the measured bf16 burst (MEASURED_PEAKS.json)
I8_PEAK_TOPS = 1664.3 * 2      # fallback: twice the measured bf16 burst (MEASURED_PEAKS.json)


def i8_peak():
    """Sustained dense int8 tcgen05 rate measured on this pool by
    tools/i8_peak.cu (profiles/i8_peak.json, the M = N = 128 shape k_oz_gram
    issues), else the 2 x bf16 fallback."""
    f = ROOT / "profiles" / "i8_peak.json"
    try:
        d = json.loads(f.read_text())
        return float(d["tops_1sm_128x128_sustained"]), (
            "sustained dense int8 rate measured by tools/i8_peak.cu on this pool (profiles/i8_peak.json: "
            "tcgen05.mma kind::i8 M=N=128 from resident smem operands, 148 SMs, ~0.3 s; the burst rate is "
            f"{d['tops_1sm_128x128']:.0f} TOPS); oz_gram runs 13 ms inside a long step")
    except Exception:  # noqa: BLE001
        return I8_PEAK_TOPS, "twice the measured bf16 burst peak of MEASURED_PEAKS.json (dense int8 = 2x bf16 rate)"


def parse_args():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--subjects", type=int, default=None, help="override the subject count (per job)")
    ap.add_argument("--e2e-fits", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--algorithm", default="auto", choices=["auto", "stream", "gram"])
    ap.add_argument("--gram-int8", default="on", choices=["on", "off"],
                    help="fp64 Gram path: X^T X from int8 slices on tcgen05 (on) or fp64 DMMA (off)")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def workload(args):
    from paper_1608_04647_b200.data import config_by_name

    cfg = config_by_name(args.config)
    if args.subjects:
        cfg["n_subjects"] = args.subjects
    return cfg


def config_json(cfg, name, world):
    b = 8 if cfg["dtype"] == "f64" else 4
    xbytes = cfg["n_subjects"] * cfg["n_voxels"] * cfg["n_trs"] * b
    return {
        "workload": (f"{name}: {cfg['n_subjects']} subjects x {cfg['n_voxels']} voxels x {cfg['n_trs']} TRs, "
                     f"k={cfg['k']}, {cfg['dtype']}, BASELINE recipe"),
        "n_subjects": cfg["n_subjects"], "n_voxels": cfg["n_voxels"], "n_trs": cfg["n_trs"], "k": cfg["k"],
        "fit_iterations": cfg["iterations"], "x_bytes": xbytes,
        "l2_policy": f"inputs larger than L2 ({xbytes / 1e9:.1f} GB of X-hat streamed per pass vs 126 MB L2)",
        "parallelism": f"subject shards x {world} ranks (contiguous, cli.py:82-85); ordered all-gather per iteration",
    }


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (STREAM copy, of measured)"
        except Exception:  # noqa: BLE001
            pass
    return FALLBACK_HBM_GBS, "B200_PROFILING.md fallback 6.65 TB/s (of fallback)"


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.proc = None
        self.path = None
        self.device_index = device_index

    def start(self):
        import torch

        ident = str(self.device_index)
        try:
            uuid = str(torch.cuda.get_device_properties(self.device_index).uuid)
            ident = uuid if uuid.startswith("GPU-") else f"GPU-{uuid}"
        except Exception:  # noqa: BLE001
            pass
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ident, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        power = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(power) if power else None}


# ---------------------------------------------------------------------------
# CPU side: the reference arithmetic (oracle port) on a bounded sample
# ---------------------------------------------------------------------------

def cpu_iterations(xs, k, n_iter, seed=0):
    """Per-iteration seconds of the reference EM (oracle port) on ``xs``."""
    from oracle import srm_oracle as orc

    xhats = [orc.center_rows(x)[0] for x in xs]
    ws = [orc.initial_mapping(xh.shape[0], k, seed, j)[0] for j, xh in enumerate(xhats)]
    rho2 = [1.0] * len(xs)
    sigma = np.eye(k)
    times = []
    for _ in range(n_iter):
        t0 = time.perf_counter()
        terms = [orc.local_term(ws[j], rho2[j], xhats[j]) for j in range(len(xs))]
        reduced, rho0 = orc.ordered_reduce(terms, rho2)
        s, _ = orc.shared_posterior(reduced, sigma, rho0)
        sigma, tr = orc.shared_covariance(sigma, rho0, s)
        for j in range(len(xs)):
            ws[j], rho2[j] = orc.subject_update(xhats[j], s, tr)
        times.append(time.perf_counter() - t0)
    return times


def sample_subjects(cfg, n, seed):
    from paper_1608_04647_b200.data import recipe_numpy

    dt = cfg["dtype"]
    xs, _, _ = recipe_numpy(cfg["n_subjects"], cfg["n_voxels"], cfg["n_trs"], cfg["k"], seed=seed,
                            smooth=cfg["smooth"], dtype=dt, first_subject=0, count=n)
    return xs


def cpu_baseline(cfg, budget_s=20.0, seed=0):
    """The reference arithmetic on the host cores; ~budget_s of CPU work."""
    xs = sample_subjects(cfg, 1, seed)
    t1 = statistics.median(cpu_iterations(xs, cfg["k"], 2, seed))  # 1 subject-iteration
    n_sub = int(max(1, min(cfg["n_subjects"], 8, budget_s / max(t1, 1e-3) / 3)))
    xs = sample_subjects(cfg, n_sub, seed)
    times = cpu_iterations(xs, cfg["k"], 3, seed)
    t = statistics.median(times)
    units = n_sub * cfg["n_voxels"] * cfg["n_trs"]
    return {
        "value": units / t, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
        "sample": (f"oracle/srm_oracle.py (numpy/OpenBLAS restatement of factorfit.srm, bit-identical on the "
                   f"golden vectors): {n_sub} of {cfg['n_subjects']} subjects, median of 3 EM iterations "
                   f"({t:.2f} s/iteration), demean+init excluded, OpenBLAS threads = all {os.cpu_count()} cores"),
    }


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    cfg = workload(args)
    xs = sample_subjects(cfg, 1, args.seed)
    t1 = statistics.median(cpu_iterations(xs, cfg["k"], 2, args.seed))
    budget = 150.0 / max(1, args.steps + args.warmup)
    n_sub = int(max(1, min(cfg["n_subjects"], budget / max(t1, 1e-3))))
    xs = sample_subjects(cfg, n_sub, args.seed)
    times = cpu_iterations(xs, cfg["k"], args.warmup + args.steps, args.seed)[args.warmup:]
    t = float(np.mean(times))
    units = n_sub * cfg["n_voxels"] * cfg["n_trs"]
    value = units / t
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic: BASELINE generative recipe (seeded numpy PCG64 stream), reference init_subject",
        "config": config_json(cfg, args.config, args.gpus), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                         "sample": (f"{n_sub} of {cfg['n_subjects']} subjects per step (one EM iteration of the "
                                    f"oracle port of factorfit.srm per step), OpenBLAS on all host cores")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1608_04647_b200 import srm
    from paper_1608_04647_b200.collectives import TorchCommunicator, shard_bounds
    from paper_1608_04647_b200.data import SubjectData, recipe_torch
    from paper_1608_04647_b200.engine import SrmEngine

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    comm = TorchCommunicator() if world > 1 else None
    cfg = workload(args)
    start, stop = shard_bounds(cfg["n_subjects"], world, rank)
    counts = [shard_bounds(cfg["n_subjects"], world, r)[1] - shard_bounds(cfg["n_subjects"], world, r)[0]
              for r in range(world)]
    n_local = stop - start
    V, T, K = cfg["n_voxels"], cfg["n_trs"], cfg["k"]
    b = 8 if cfg["dtype"] == "f64" else 4

    xs, _, _ = recipe_torch(cfg["n_subjects"], V, T, K, seed=args.seed, smooth=cfg["smooth"],
                            dtype=cfg["dtype"], first_subject=start, count=n_local, device=dev)
    torch.cuda.synchronize()

    # ---------------- value: X resident in HBM, a K-iteration fit timed --------
    # The timed region is everything a fit does after demean + init (the
    # reference's per-iteration accounting also excludes those): the Gram
    # precompute when the Gram path is chosen, K EM iterations, and the final
    # W_i = A_i M_i.  One-time work is therefore charged to the K steps.
    algo = args.algorithm
    use_i8 = args.gram_int8 == "on"
    if algo == "auto":
        algo = srm.choose_algorithm([V] * cfg["n_subjects"], T, K, args.steps,
                                    torch.cuda.mem_get_info(dev)[0] * world, storage=cfg["dtype"],
                                    gram_int8=use_i8)
    total_iters = max(args.warmup, args.steps) + 8
    eng = SrmEngine([V] * n_local, T, K, total_iters, storage=cfg["dtype"], world_size=world, rank=rank,
                    counts=counts, ordered=True, gram=(algo == "gram"), tc=(cfg["dtype"] == "f32"),
                    gram_i8=(algo == "gram" and use_i8), device=dev)
    use_i8 = eng.gram_i8
    eng.load(xs)
    use_graph = world == 1

    def schedule(n_iter, timed_events=None):
        if timed_events:
            timed_events[0].record(torch.cuda.current_stream())
        eng.prepare_gram()
        for it in range(n_iter):
            if use_graph and eng._graph is not None:
                eng.replay()
            else:
                eng.step(comm)
                if use_graph and it == 0:
                    eng.capture()
        eng.finalize()
        if timed_events:
            timed_events[1].record(torch.cuda.current_stream())

    eng.init_mapping(args.seed, start)
    schedule(max(1, args.warmup))          # warm-up fit: configures kernels, captures the graph
    eng.raise_status()
    eng.reset()
    eng.init_mapping(args.seed, start)     # fresh EM start (untimed, like the reference's init)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    schedule(args.steps, (e0, e1))
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    eng.raise_status()
    units = cfg["n_subjects"] * V * T
    value = units / (ms / 1e3)
    tc = cfg["dtype"] == "f32"

    # per-kernel durations (CUDA events on the launch stream, untimed pass)
    st = torch.cuda.current_stream()
    prof_iter = {}
    for _ in range(5):
        one = {}
        for name, t_ms in eng.profile_iteration():  # a stage may run once per subject half
            one[name] = one.get(name, 0.0) + t_ms
        for name, t_ms in one.items():
            prof_iter.setdefault(name, []).append(t_ms)
    prof_iter = {k_: float(np.mean(v_)) for k_, v_ in prof_iter.items()}
    once = {}
    if algo == "gram":
        prof_g = {}
        for _ in range(3):
            for name, t_ms in eng.profile_gram():
                prof_g.setdefault(name, []).append(t_ms)
        once.update({k_: float(np.mean(v_)) for k_, v_ in prof_g.items()})
    prof_f = {}
    for _ in range(3):
        for name, t_ms in eng.profile_finalize():
            prof_f.setdefault(name, []).append(t_ms)
    once.update({k_: float(np.mean(v_)) for k_, v_ in prof_f.items()})
    eng.raise_status()
    # kernels of the timed region: every stage is one launch except oz_split
    # (column maxima + slicing)
    launches = (eng.launches_per_iteration * args.steps + len(prof_f)
                + (len(prof_g) + ("oz_split" in prof_g) if algo == "gram" else 0))
    del eng
    torch.cuda.empty_cache()

    # time share of each kernel inside the timed region (K iterations + one-time work)
    region_ms = {k_: v_ * args.steps for k_, v_ in prof_iter.items()}
    region_ms.update(once)
    tot = sum(region_ms.values())
    step_share = {k_: v_ / tot for k_, v_ in region_ms.items()}
    dom = max(region_ms, key=region_ms.get)
    hbm_peak, peak_src = peaks()
    local_units = n_local * V * T
    ldx = -(-T // 32) * 32
    nt = -(-ldx // 128)
    if dom in ("gram_tiles", "oz_gram"):
        launch_ms = once[dom]
        alg_flops = float(n_local) * V * T * (T + 1)          # symmetric X^T X: T(T+1)/2 dots of length V
        alg_bytes = float(local_units * b)                      # X-hat read once
        # int8 products issued by oz_gram per upper 128 x 128 tile and 32-voxel block: the slice
        # pairs s + s' < 7 (28 for fp64's 7 slices; all 16 for fp32's 4)
        products = 28 if cfg["dtype"] == "f64" else 16
        i8_ops = 2.0 * products * nt * (nt + 1) / 2 * 128 * 128 * (-(-V // 32) * 32) * n_local
    elif dom in ("final_a", "oz_w", "apply_w"):
        launch_ms = once[dom]
        alg_flops = 2.0 * local_units * K
        alg_bytes = float(local_units * b)
    else:
        launch_ms = prof_iter[dom]
        if dom in ("contract_a", "contract_e_xhat", "tc_apass", "tc_bpass"):
            alg_flops = 2.0 * local_units * K                   # one pass: 2K flops per unit
            alg_bytes = float(local_units * b)                  # b bytes per unit per pass
        else:
            alg_flops = 2.0 * n_local * K * T * T
            alg_bytes = float(n_local * T * T * 8)
    achieved_tf = alg_flops / (launch_ms / 1e3) / 1e12
    achieved_gbs = alg_bytes / (launch_ms / 1e3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get(f"{args.config}:{algo}", {}).get(dom)
        except Exception:  # noqa: BLE001
            traffic = None
    if dom == "oz_gram":
        achieved_tops = i8_ops / (launch_ms / 1e3) / 1e12
        i8_pk, i8_src = i8_peak()
        roofline = {
            "bound": "tensor", "achieved": achieved_tops, "peak": i8_pk, "unit": "TOPS (int8)",
            "frac": achieved_tops / i8_pk, "traffic": traffic, "kernel": dom, "launch_ms": launch_ms,
            "algorithmic_int8_ops_per_launch": i8_ops, "algorithmic_flops_per_launch": alg_flops,
            "algorithmic_bytes_per_launch": alg_bytes, "peak_source": i8_src,
        }
        other_roofline = {
            "bound": "fp64-equivalent", "achieved": achieved_tf, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved_tf / DMMA_PEAK_TFLOPS, "kernel": dom,
            "peak_source": "X^T X flops (V T (T+1)) per second against the measured fp64 DMMA peak (37.1 TF/s)",
        }
    elif dom in ("tc_apass", "tc_bpass"):
        # fp32 X-hat on tcgen05 (3xTF32): the pass is designed to be HBM-bound
        roofline = {
            "bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved_gbs / hbm_peak, "traffic": traffic, "kernel": dom, "launch_ms": launch_ms,
            "algorithmic_bytes_per_launch": alg_bytes, "algorithmic_flops_per_launch": alg_flops,
            "peak_source": peak_src,
        }
        other_roofline = {
            "bound": "tensor (3xTF32 tcgen05)", "achieved": 3 * achieved_tf, "peak": TF32_PEAK_TFLOPS,
            "unit": "TFLOP/s", "frac": 3 * achieved_tf / TF32_PEAK_TFLOPS, "kernel": dom,
            "peak_source": "half the measured bf16 burst peak of MEASURED_PEAKS.json (tf32 = 1/2 bf16 rate)",
        }
    else:
        roofline = {
            "bound": "tensor", "achieved": achieved_tf, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved_tf / DMMA_PEAK_TFLOPS, "traffic": traffic, "kernel": dom, "launch_ms": launch_ms,
            "algorithmic_flops_per_launch": alg_flops, "algorithmic_bytes_per_launch": alg_bytes,
            "peak_source": ("FP64 tensor pipe (mma.sync.m8n8k4.f64 = SASS DMMA) measured on this pool by "
                            "tools/fp64_peak.cu (37.1 TF/s); the path computes in fp64 like the reference, "
                            "so the bf16 figure of MEASURED_PEAKS.json does not apply"),
        }
        other_roofline = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                          "frac": achieved_gbs / hbm_peak, "kernel": dom, "peak_source": peak_src}
    prof = {"per_iteration_ms": prof_iter, "one_time_ms": once}

    # ---------------- e2e: public API, pinned host inputs ---------------------
    e2e = None
    if not args.no_e2e:
        host = [x.to("cpu").pin_memory() for x in xs]
        del xs
        torch.cuda.empty_cache()
        subjects = [SubjectData(f"sub-{start + j:04d}", host[j]) for j in range(n_local)]
        conf = srm.SrmConfig(k=K, iterations=cfg["iterations"], seed=args.seed)
        srm.fit(subjects, conf, comm, algorithm=args.algorithm, gram_int8=args.gram_int8 == "on")  # warm-up (allocator, kernels)
        times = []
        for _ in range(max(1, args.e2e_fits)):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            model = srm.fit(subjects, conf, comm, algorithm=args.algorithm, gram_int8=args.gram_int8 == "on")
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if world > 1:
                tt = torch.tensor([dt], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt = float(tt.item())
            times.append(dt)
        dt = min(times)
        h2d = cfg["n_subjects"] * V * T * b
        d2h = cfg["n_subjects"] * V * (K + 1) * 8 + K * T * 8 + K * K * 8
        e2e = {"value": units * cfg["iterations"] / dt, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "seconds_per_fit": dt,
               "step": (f"one srm.fit call ({cfg['iterations']} EM iterations) on pinned host arrays: H2D, "
                        "demean, PCG64 init + device polar, EM loop, model read-back")}
        del model

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, seed=args.seed)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": cfg["dtype"],
            "data": "synthetic: BASELINE generative recipe (seeded, device Philox stream); reference init",
            "config": config_json(cfg, args.config, world),
            "roofline": roofline, "secondary_roofline": other_roofline, "algorithm": algo,
            "gram_xtx": (("int8 slices on tcgen05 (7 slices, ~2^-48 of column max)" if cfg["dtype"] == "f64"
                          else "int8 slices on tcgen05 (4 slices, ~2^-27 of column max; fp32 data)")
                         if use_i8 else "fp64 DMMA")
            if algo == "gram" else None,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "kernel_ms": prof, "kernel_share": step_share, "impl": "ours",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
