#!/usr/bin/env python
"""Benchmark of the SRM EM fit on B200 (BASELINE.json metric and config).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
    python bench.py --impl reference ...      # the reference CPU arithmetic

A *step* is one complete fit of the config's fixed EM iteration count
(BASELINE.json: 10 / 20 / 10 / 10 / 5 for cfg 1-5; srm.py:254-287) with
X-hat already resident in HBM: the device part of the initialisation (the
srm.py:101-118 polar of the PCG64 draw and the first E-step term), the
one-time Gram precompute when that path is chosen, the EM iterations and
the final W_i (srm.py:315-327).  Demean and the host PCG64 draw are not in
it (the reference's own per-iteration accounting also excludes them).
``value`` is the whole-job subject*voxel*TR/s per EM iteration:
n_subjects * V * T * iterations / (step seconds), timed with CUDA events
over exactly K steps (max over ranks).  ``e2e`` is the same metric through
the public API ``srm.fit`` on pinned host arrays: host-to-device copies,
demean, the reference initialisation and the read-back of the model
included.  The default workload is BASELINE config 2 (40 subjects x 30,000
voxels x 1,000 TRs, k=50, fp64, 20 iterations); subjects are sharded across
ranks (strong scaling, cli.py:82-85 contiguous shards).

Under torchrun (N > 1) every rank drives one GPU over NCCL; the per-iteration
exchange is the ordered column-block exchange (an all-to-all of the E-step
terms in N TR blocks, ordered block sums, an all-gather of K x T / N),
captured with the iteration in one CUDA graph per rank.
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
    ap.add_argument("--steps", type=int, default=10)
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
        "parallelism": (f"subject shards x {world} ranks (contiguous, cli.py:82-85); ordered column-block "
                        "exchange per iteration (all-to-all + all-gather of K x T / N)"),
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

def cpu_iterations(xs, k, n_iter, seed=0, threads=None):
    """Per-iteration seconds of the reference EM (oracle port) on ``xs``.

    The step functions keep the reference's cost structure (srm.py:116-155:
    four passes over X-hat per subject-iteration and the V x K SVD);
    ``threads`` caps the BLAS threads (OPENBLAS_NUM_THREADS, via threadpoolctl).
    """
    from threadpoolctl import threadpool_limits

    from oracle import srm_oracle as orc

    with threadpool_limits(limits=threads):
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


def _proc_worker(xs, k, n_iter, seed, threads, barrier, out):
    out.put(cpu_iterations_sync(xs, k, n_iter, seed, threads, barrier))


def cpu_iterations_sync(xs, k, n_iter, seed, threads, barrier):
    """cpu_iterations on one worker's share with a barrier per iteration
    (the reference's sockets backend synchronises at its gather/broadcast)."""
    from threadpoolctl import threadpool_limits

    from oracle import srm_oracle as orc

    with threadpool_limits(limits=threads):
        xhats = [orc.center_rows(x)[0] for x in xs]
        ws = [orc.initial_mapping(xh.shape[0], k, seed, j)[0] for j, xh in enumerate(xhats)]
        rho2 = [1.0] * len(xs)
        sigma = np.eye(k)
        times = []
        for _ in range(n_iter):
            barrier.wait()
            t0 = time.perf_counter()
            terms = [orc.local_term(ws[j], rho2[j], xhats[j]) for j in range(len(xs))]
            reduced, rho0 = orc.ordered_reduce(terms, rho2)  # this worker's share only (timing model)
            s, _ = orc.shared_posterior(reduced, sigma, rho0)
            sigma, tr = orc.shared_covariance(sigma, rho0, s)
            for j in range(len(xs)):
                ws[j], rho2[j] = orc.subject_update(xhats[j], s, tr)
            barrier.wait()
            times.append(time.perf_counter() - t0)
    return times


def cpu_process_iterations(xs, k, n_iter, seed, procs):
    """The paper's best CPU mode (cli.py:113-200 ``--backend sockets
    --spawn-local P``): P forked workers with cores / P BLAS
    threads each and contiguous subject shards; per-iteration time is the
    barrier-to-barrier time (the K x T exchange, ~KT bytes, is not modelled)."""
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    cores = os.cpu_count() or 1
    barrier = ctx.Barrier(procs)
    out = ctx.Queue()
    shares = [xs[i * len(xs) // procs:(i + 1) * len(xs) // procs] for i in range(procs)]
    ps = [ctx.Process(target=_proc_worker, args=(sh, k, n_iter, seed, max(1, cores // procs), barrier, out))
          for sh in shares]
    for p in ps:
        p.start()
    res = [out.get() for _ in ps]
    for p in ps:
        p.join()
    return [max(r[i] for r in res) for i in range(n_iter)]


def blas_info():
    try:
        from threadpoolctl import threadpool_info

        libs = [f"{d.get('internal_api')} {d.get('version')}" for d in threadpool_info() if d.get("user_api") == "blas"]
    except Exception:  # noqa: BLE001
        libs = []
    model = ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"blas": ", ".join(libs) or "unknown", "cpu": model, "cores": os.cpu_count()}


def sample_subjects(cfg, n, seed, device_xs=None):
    """The first ``n`` subjects of the workload as host arrays -- the same
    bytes the GPU arm fits (device Philox stream copied to the host) when a
    GPU is present, else the host generator's stream."""
    if device_xs is not None:
        return [np.ascontiguousarray(x.cpu().numpy()) for x in device_xs[:n]]
    try:
        import torch

        if torch.cuda.is_available():
            from paper_1608_04647_b200.data import recipe_torch

            out = []
            for i in range(n):
                x, _, _ = recipe_torch(cfg["n_subjects"], cfg["n_voxels"], cfg["n_trs"], cfg["k"], seed=seed,
                                       smooth=cfg["smooth"], dtype=cfg["dtype"], first_subject=i, count=1)
                out.append(x[0].cpu().numpy())
            return out
    except Exception:  # noqa: BLE001
        pass
    from paper_1608_04647_b200.data import recipe_numpy

    xs, _, _ = recipe_numpy(cfg["n_subjects"], cfg["n_voxels"], cfg["n_trs"], cfg["k"], seed=seed,
                            smooth=cfg["smooth"], dtype=cfg["dtype"], first_subject=0, count=n)
    return xs


def cpu_baseline(cfg, host_xs, budget_s=24.0, seed=0):
    """The reference arithmetic on the host cores, swept over
    OPENBLAS_NUM_THREADS in {1, cores/2, cores} and P-process shards
    (BASELINE.md section 3); ~budget_s of CPU work in total."""
    cores = os.cpu_count() or 1
    t1 = statistics.median(cpu_iterations(host_xs[:1], cfg["k"], 2, seed))  # 1 subject-iteration, all threads
    n_sub = int(max(1, min(len(host_xs), cfg["n_subjects"], budget_s / 8 / max(t1, 1e-3))))
    xs = host_xs[:n_sub]
    units = n_sub * cfg["n_voxels"] * cfg["n_trs"]
    sweep = {}
    for th in sorted({1, max(1, cores // 2), cores}):
        sweep[f"1 proc x {th} threads"] = units / statistics.median(cpu_iterations(xs, cfg["k"], 2, seed, th))
    for procs in sorted({min(n_sub, 4), min(n_sub, cores)}):
        if procs > 1:
            sweep[f"{procs} procs x {max(1, cores // procs)} threads"] = units / statistics.median(
                cpu_process_iterations(xs, cfg["k"], 2, seed, procs))
    best = max(sweep, key=sweep.get)
    info = blas_info()
    return {
        "value": sweep[best], "unit": UNIT, "cores": cores, "kind": "port",
        "sample": (f"oracle/srm_oracle.py (numpy/scipy restatement of factorfit.srm with its cost structure, "
                   f"bit-identical on the golden vectors): {n_sub} of {cfg['n_subjects']} subjects (the same bytes "
                   f"as the GPU arm), median of 2 EM iterations per setting, demean + init excluded; best setting "
                   f"{best}"),
        "sweep": sweep, "blas": info["blas"], "cpu": info["cpu"],
    }


def run_reference(args):
    """The reference's CPU arithmetic (oracle port, the reference's cost
    structure) in its best host configuration: one process with all BLAS
    threads, or P processes x cores / P threads (the paper's sockets
    spawn-local mode), whichever a one-iteration probe finds faster."""
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    cfg = workload(args)
    cores = os.cpu_count() or 1
    xs1 = sample_subjects(cfg, 1, args.seed)
    t1 = statistics.median(cpu_iterations(xs1, cfg["k"], 2, args.seed))
    budget = 150.0 / max(1, args.steps + args.warmup)
    procs = min(cfg["n_subjects"], 8, cores)
    n_sub = int(max(procs, min(cfg["n_subjects"], budget / max(t1, 1e-3))))
    xs = sample_subjects(cfg, n_sub, args.seed)
    probe = {1: statistics.median(cpu_iterations(xs, cfg["k"], 1, args.seed))}
    if procs > 1:
        probe[procs] = statistics.median(cpu_process_iterations(xs, cfg["k"], 1, args.seed, procs))
    best = min(probe, key=probe.get)
    n_iter = args.warmup + args.steps
    if best == 1:
        times = cpu_iterations(xs, cfg["k"], n_iter, args.seed)[args.warmup:]
        mode = f"1 process x {cores} BLAS threads"
    else:
        times = cpu_process_iterations(xs, cfg["k"], n_iter, args.seed, best)[args.warmup:]
        mode = f"{best} processes x {max(1, cores // best)} BLAS threads (sockets spawn-local mode)"
    t = float(np.mean(times))
    units = n_sub * cfg["n_voxels"] * cfg["n_trs"]
    value = units / t
    info = blas_info()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic: BASELINE generative recipe (device Philox stream copied to the host: the GPU arm's bytes), "
                "reference init_subject",
        "config": config_json(cfg, args.config, args.gpus), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": (f"{n_sub} of {cfg['n_subjects']} subjects per step (one EM iteration of the "
                                    f"oracle port of factorfit.srm per step); {mode}, the faster of the probed "
                                    f"host configurations {{{', '.join(f'{p} proc: {v:.2f} s' for p, v in probe.items())}}}"),
                         "blas": info["blas"], "cpu": info["cpu"]},
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
    # SRM_BENCH_BACKEND=gloo with SRM_BENCH_ONE_GPU=1 runs every rank on GPU 0
    # with the exchange through host memory: a check of the multi-rank flow on a
    # one-GPU box (no kernel waits on another rank's), not a scaling measurement
    backend = os.environ.get("SRM_BENCH_BACKEND", "nccl")
    gpu = 0 if os.environ.get("SRM_BENCH_ONE_GPU") == "1" else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    comm = TorchCommunicator() if world > 1 else None
    cfg = workload(args)
    iters = cfg["iterations"]
    start, stop = shard_bounds(cfg["n_subjects"], world, rank)
    counts = [shard_bounds(cfg["n_subjects"], world, r)[1] - shard_bounds(cfg["n_subjects"], world, r)[0]
              for r in range(world)]
    n_local = stop - start
    V, T, K = cfg["n_voxels"], cfg["n_trs"], cfg["k"]
    b = 8 if cfg["dtype"] == "f64" else 4

    xs, _, _ = recipe_torch(cfg["n_subjects"], V, T, K, seed=args.seed, smooth=cfg["smooth"],
                            dtype=cfg["dtype"], first_subject=start, count=n_local, device=dev)
    torch.cuda.synchronize()

    # ---------------- value: X-hat resident in HBM, K complete fits timed ------
    algo = args.algorithm
    use_i8 = args.gram_int8 == "on"
    if algo == "auto":  # the choice srm.fit makes for this config at its iteration count
        algo = srm.choose_algorithm([V] * cfg["n_subjects"], T, K, iters,
                                    torch.cuda.mem_get_info(dev)[0] * world, storage=cfg["dtype"],
                                    gram_int8=use_i8)
    eng = SrmEngine([V] * n_local, T, K, iters, storage=cfg["dtype"], world_size=world, rank=rank,
                    counts=counts, ordered=True, colblock=world > 1 and hasattr(comm, "all_to_all_into"),
                    gram=(algo == "gram"), tc=(cfg["dtype"] == "f32"),
                    gram_i8=(algo == "gram" and use_i8), device=dev)
    use_i8 = eng.gram_i8
    eng.load(xs)
    # the same bytes on the host: pinned for the e2e fits, the first subjects for the CPU baseline
    host = None
    if not args.no_e2e:
        host = [x.to("cpu").pin_memory() for x in xs]
    cpu_xs = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_xs = [x.cpu().numpy() for x in xs[:8]]
    del xs
    torch.cuda.empty_cache()
    use_graph = world == 1
    # N > 1 over NCCL: {all-gather / all-reduce, E-step, M-step} as one graph per rank
    use_xgraph = world > 1 and eng.exchange_capturable(comm)
    eng.prepare_gram()
    eng.init_mapping(args.seed, start)  # the host PCG64 draws (srm.py:111), uploaded once
    draws = eng.amat.clone()            # each step restarts from them: only device work is timed
    # the int8 Gram path only reads the draws (the per-iteration A_i never
    # lands in AMAT), so a step need not restore them -- checked after the
    # warm-up steps, restored every step otherwise
    restore = [not eng.gram_i8]

    def step():
        # one complete fit: restart, one-time Gram (its X-hat slices also feed the
        # init term), device init (polar of the draw, first E-step term), the
        # config's EM iterations, final W
        eng.reset()
        if restore[0]:
            eng.amat.copy_(draws)
        eng.prepare_gram()
        eng.init_kernels()
        for _ in range(iters):
            if use_graph and eng._graph is not None:
                eng.replay()
            elif use_xgraph and eng._xgraph is not None:
                eng.replay_exchange()
            else:
                eng.step(comm)
                if use_graph:
                    eng.capture()
                elif use_xgraph:
                    eng.capture_exchange(comm)  # after one eager exchange
        eng.finalize()

    for _ in range(max(1, args.warmup)):  # configures kernels, captures the iteration graph
        step()
    eng.raise_status()
    if not restore[0] and not torch.equal(eng.amat, draws):
        restore[0] = True  # something wrote AMAT: restore the draws every step
        step()
    if not restore[0]:
        del draws
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(gpu)
    sampler.start()
    time.sleep(0.2)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
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
    value = units * iters / (ms / 1e3)

    # per-kernel durations (CUDA events on the launch stream, untimed passes)
    prof_iter = {}
    for _ in range(5):
        one = {}
        for name, t_ms in eng.profile_iteration():  # a stage may run once per subject half
            one[name] = one.get(name, 0.0) + t_ms
        for name, t_ms in one.items():
            prof_iter.setdefault(name, []).append(t_ms)
    prof_iter = {k_: float(np.mean(v_)) for k_, v_ in prof_iter.items()}
    once = {}
    prof_g = {}
    if algo == "gram":
        for _ in range(3):
            for name, t_ms in eng.profile_gram():
                prof_g.setdefault(name, []).append(t_ms)
        once.update({k_: float(np.mean(v_)) for k_, v_ in prof_g.items()})
        if "oz_gram_pairs" in once:  # SRM_B200_GRAM_PAIRS=1: the CTA-pair tiles are part of the Gram
            once["oz_gram"] = once.get("oz_gram", 0.0) + once.pop("oz_gram_pairs")
    prof_f = {}
    for _ in range(3):
        for name, t_ms in eng.profile_finalize():
            prof_f.setdefault(name, []).append(t_ms)
    once.update({k_: float(np.mean(v_)) for k_, v_ in prof_f.items()})
    eng.raise_status()
    # kernels of one step: reset + the init kernels (6; 9 with the int8 init
    # term: draw column maxima, draw slices, G^T Xhat), the Gram stages, the
    # iterations, the final W
    init_launches = 10 if use_i8 else 7
    per_step = (init_launches + (len(prof_g) if algo == "gram" else 0)
                + eng.launches_per_iteration * iters + len(prof_f))
    launches = per_step * args.steps
    del eng
    torch.cuda.empty_cache()

    # time share of each kernel inside one step (iterations x per-iteration + one-time)
    region_ms = {k_: v_ * iters for k_, v_ in prof_iter.items()}
    region_ms.update(once)
    tot = sum(region_ms.values())
    step_share = {k_: v_ / tot for k_, v_ in region_ms.items()}
    dom = max(region_ms, key=region_ms.get)
    hbm_peak, peak_src = peaks()
    local_units = n_local * V * T
    ldx = -(-T // 32) * 32
    nt = -(-ldx // 128)
    slice_b = 8 if cfg["dtype"] == "f64" else 4  # int8 slice bytes per X-hat value (7 or 4 slices, padded)
    if dom in ("gram_tiles", "oz_gram"):
        launch_ms = once[dom]
        alg_flops = float(n_local) * V * T * (T + 1)          # symmetric X^T X: T(T+1)/2 dots of length V
        alg_bytes = float(local_units * (slice_b if dom == "oz_gram" else b))
        # int8 products per Gram entry and 32-voxel block off the diagonal tiles: the slice pairs
        # s + s' <= 6 (28 of fp64's 7 slices) or <= 3 (10 of fp32's 4; the diagonal tiles'
        # extra d-groups are not counted); useful = T(T+1)/2 entries
        products = 28 if cfg["dtype"] == "f64" else 10
        i8_ops = 2.0 * products * (T * (T + 1) / 2) * (-(-V // 32) * 32) * n_local
    elif dom in ("final_a", "oz_w", "apply_w"):
        launch_ms = once[dom]
        alg_flops = 2.0 * local_units * K
        alg_bytes = float(local_units * (slice_b if dom == "oz_w" else b))
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
            "work": "useful slice products only: T(T+1)/2 Gram entries per subject (the padded 128 x 128 "
                    "diagonal tiles and the mirrored half are not counted)",
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
    # the metric's HBM half: every kernel that streams X-hat (or its int8 slices), at its
    # algorithmic bytes per launch (reads of X-hat / slices once, writes of slices / W once)
    xk_bytes = {
        "oz_split": local_units * (b + slice_b),                   # read X-hat, write the slices
        "oz_gram": local_units * slice_b,                          # read the slices once
        "oz_w": local_units * slice_b + n_local * V * K * 8,       # read the slices, write W
        "gram_tiles": local_units * b,
        "final_a": local_units * b + n_local * V * (-(-K // 8) * 8) * 8,
        "contract_a": local_units * b + n_local * V * (-(-K // 8) * 8) * 8,
        "contract_e_xhat": local_units * b,
        "tc_apass": local_units * b, "tc_bpass": local_units * b,
    }
    per_kernel = {}
    for name, nbytes in xk_bytes.items():
        t_ms = once.get(name, prof_iter.get(name))
        if t_ms:
            gbs = nbytes / (t_ms / 1e3) / 1e9
            per_kernel[name] = {"bytes": nbytes, "ms": t_ms, "achieved": gbs, "frac": gbs / hbm_peak,
                                "per": "launch" if name in once else "iteration"}
    x_read = 2.0 * b * units * iters  # two X-hat reads per subject-iteration
    roofline_hbm = {
        "unit": "GB/s", "peak": hbm_peak, "peak_source": peak_src, "kernels": per_kernel,
        "streaming_equivalent": {
            "achieved": x_read / (ms / 1e3) / 1e9, "frac": x_read / (ms / 1e3) / 1e9 / hbm_peak,
            "note": ("SURVEY.md §8(d) algorithmic bytes (2 X-hat reads per subject-iteration) over the step "
                     "time; above 1 where the Gram path replaces the per-iteration passes"),
        },
    }
    prof = {"per_iteration_ms": prof_iter, "one_time_ms": once}

    # ---------------- e2e: public API, pinned host inputs ---------------------
    e2e = None
    if host is not None:
        subjects = [SubjectData(f"sub-{start + j:04d}", host[j]) for j in range(n_local)]
        conf = srm.SrmConfig(k=K, iterations=iters, seed=args.seed)
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
        e2e = {"value": units * iters / dt, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "seconds_per_fit": dt,
               "step": (f"one srm.fit call ({iters} EM iterations) on pinned host arrays: H2D, "
                        "demean, PCG64 init + device polar, EM loop, model read-back")}
        del model

    cpu = None
    if cpu_xs is not None:
        cpu = cpu_baseline(cfg, cpu_xs, seed=args.seed)

    if rank == 0:
        conf_json = config_json(cfg, args.config, world)
        conf_json["step"] = (f"one complete fit from HBM-resident X-hat: device init, "
                             f"{'one-time int8 X^T X, ' if algo == 'gram' else ''}{iters} EM iterations, final W")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": cfg["dtype"],
            "data": "synthetic: BASELINE generative recipe (seeded, device Philox stream); reference init",
            "config": conf_json,
            "roofline": roofline, "secondary_roofline": other_roofline, "roofline_hbm": roofline_hbm,
            "algorithm": algo,
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
