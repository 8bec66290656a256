"""Command line for the B200 SRM fit: the reference's ``fit-srm`` and ``bench``.

    python -m paper_1608_04647_b200 fit-srm --manifest M --k K --iters N --out DIR
    python -m paper_1608_04647_b200 bench   --manifest M --k K --iters N [--out DIR]

Same arguments, artifacts and report schema as ``factorfit.cli``
(``/root/reference/pkg/src/factorfit/cli.py:64-102, 214-263, 381-423``):

* ``fit-srm`` writes ``subjects/{id}_mapping.sfab`` (W_i), ``{id}_mean.sfab``
  (mu_i as V x 1), and on rank 0 ``shared_response.sfab`` (S),
  ``shared_covariance.sfab`` (Sigma_s), ``noise_variance.sfab`` (rho^2 of all
  subjects, N x 1) and ``report.json``;
* ``bench`` prints the report (and writes it with ``--out``).

The report keeps the reference keys (``schema``, ``command``, ``backend``,
``workers``, ``timings`` {load, compute, communicate}, ``objective``,
``flops`` -- the reference's analytic estimate, cli.py:66-80 --,
``gflops_per_s``, ``outputs``) and adds a ``device`` object: GPU name, the
fit's per-phase device-synchronised seconds and the achieved X-hat bytes per
second of the EM iterations.

Backends: ``serial`` (one process, one GPU) and ``nccl`` (one process per GPU
under torchrun, ``TorchCommunicator``).  Subjects are split into contiguous
per-rank shards (cli.py:82-85).  Exit codes: 0 success, 1 runtime or data
error (a JSON error object on stderr), 2 usage error.
"""

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

from .errors import FactorFitError

REPORT_SCHEMA = 1


class UsageError(FactorFitError):
    """Bad command-line arguments (exit code 2)."""


def srm_flops_per_subject_iteration(n_voxels, n_trs, k):
    """The reference's analytic flop count of one subject-iteration (cli.py:66-75):
    two V x T x K products, one V x K x K product and a V x K economy SVD
    counted as a Householder QR."""
    v, t, k = float(n_voxels), float(n_trs), float(k)
    return 2.0 * (2.0 * v * t * k) + 2.0 * v * k * k + (2.0 * v * k * k - (2.0 / 3.0) * k ** 3)


def srm_flop_estimate(voxel_counts, n_trs, k, iterations):
    return float(iterations) * sum(srm_flops_per_subject_iteration(v, n_trs, k) for v in voxel_counts)


def make_report(command, backend, workers, timings, objective, flops, outputs, device=None):
    """The reference report (cli.py:88-102) plus a ``device`` object."""
    timings = {k: max(float(v), 0.0) for k, v in timings.items()}
    compute = timings.get("compute", 0.0)
    gflops = flops / compute / 1e9 if compute > 0.0 and flops > 0.0 else 0.0
    rep = {
        "schema": REPORT_SCHEMA,
        "command": command,
        "backend": backend,
        "workers": workers,
        "timings": timings,
        "objective": [float(x) for x in objective],
        "flops": float(flops),
        "gflops_per_s": float(gflops),
        "outputs": outputs,
    }
    if device is not None:
        rep["device"] = device
    return rep


def write_report(out_dir, report):
    path = Path(out_dir) / "report.json"
    with open(path, "w") as fh:
        json.dump(report, fh, indent=2)
        fh.write("\n")
    return path


def _communicator(backend):
    from .collectives import SerialCommunicator, TorchCommunicator

    if backend == "serial":
        return SerialCommunicator()
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return TorchCommunicator()


def _fit(args, command):
    from . import data_io, srm

    if args.k < 1:
        raise UsageError("--k must be at least 1")
    if args.iters < (1 if command == "fit-srm" else 0):
        raise UsageError("--iters must be at least 1" if command == "fit-srm" else "--iters must be nonnegative")
    manifest = data_io.load_manifest(args.manifest, model="srm")
    headers = [data_io.read_header(e.data_path) for e in manifest.subjects]
    n_trs = headers[0][1]
    flops = srm_flop_estimate([h[0] for h in headers], n_trs, args.k, args.iters)
    out_dir = Path(args.out) if args.out else None
    comm = _communicator(args.backend)
    if out_dir is not None and comm.rank == 0:
        out_dir.mkdir(parents=True, exist_ok=True)
        if command == "fit-srm":
            (out_dir / "subjects").mkdir(exist_ok=True)
    comm.barrier()
    import torch

    t0 = time.perf_counter()
    phases = {}
    objective = []
    model = None
    subjects = data_io.open_subjects(manifest, comm.rank, comm.size, threads=args.read_threads)
    if args.iters > 0:
        config = srm.SrmConfig(k=args.k, iterations=args.iters, seed=args.seed)
        model = srm.fit(subjects, config, comm, timings=phases, algorithm=args.algorithm)
        objective = model.objective_trace
    else:
        for s in subjects:
            s.X.result()
    torch.cuda.synchronize()
    comm.barrier()
    t1 = time.perf_counter()
    if command == "fit-srm" and model is not None:
        for sid, W, mu in zip(model.subject_ids, model.W, model.mu):
            data_io.save_matrix(out_dir / "subjects" / f"{sid}_mapping.sfab", W)
            data_io.save_matrix(out_dir / "subjects" / f"{sid}_mean.sfab", np.asarray(mu)[:, None])
        if comm.rank == 0:
            data_io.save_matrix(out_dir / "shared_response.sfab", model.S)
            data_io.save_matrix(out_dir / "shared_covariance.sfab", model.sigma_s)
            data_io.save_matrix(out_dir / "noise_variance.sfab", np.asarray(model.rho2_all)[:, None])
    if comm.rank != 0:
        return 0
    comm_time = float(getattr(comm.stats, "seconds", 0.0))
    # the reference's "load" is reading the subject files; here the reads stream
    # into the fit's upload pipeline, so load = setup + upload/demean phases
    load = phases.get("setup", 0.0) + phases.get("load", 0.0)
    timings = {"load": load, "compute": (t1 - t0) - load - comm_time, "communicate": comm_time}
    x_bytes = sum(h[0] for h in headers) * n_trs * 8
    em = phases.get("em", 0.0)
    device = {
        "name": torch.cuda.get_device_name(),
        "gpus": comm.size,
        "phases_s": {k: float(v) for k, v in phases.items()},
        "x_hat_bytes": int(x_bytes),
        "em_iterations": len(objective),
        "em_s_per_iteration": em / max(len(objective), 1),
    }
    report = make_report(command, args.backend, comm.size, timings, objective, flops,
                         {"dir": str(out_dir)} if (command == "fit-srm" and out_dir) else {}, device)
    if command == "bench":
        print(json.dumps(report, indent=2))
    if out_dir is not None:
        write_report(out_dir, report)
    return 0


def build_parser():
    ap = argparse.ArgumentParser(prog="python -m paper_1608_04647_b200",
                                 description="B200 SRM fit (factorfit fit-srm / bench)")
    sub = ap.add_subparsers(dest="command", required=True)
    for name in ("fit-srm", "bench"):
        p = sub.add_parser(name)
        p.add_argument("--manifest", required=True)
        p.add_argument("--k", type=int, required=True)
        p.add_argument("--iters", type=int, default=10)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--out", required=(name == "fit-srm"), default=None)
        p.add_argument("--backend", choices=["serial", "nccl"], default="serial")
        p.add_argument("--algorithm", choices=["auto", "stream", "gram"], default="auto")
        p.add_argument("--read-threads", type=int, default=8)
    return ap


def main(argv=None):
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return int(e.code or 0)
    try:
        return _fit(args, args.command)
    except UsageError as e:
        print(json.dumps({"error": "UsageError", "message": str(e)}), file=sys.stderr)
        return 2
    except (FactorFitError, OSError, ValueError, KeyError) as e:
        err = {"error": type(e).__name__, "message": str(e)}
        for attr in ("offenders", "field", "offset", "pivot", "rank"):
            if getattr(e, attr, None) is not None:
                err[attr] = getattr(e, attr)
        print(json.dumps(err), file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
