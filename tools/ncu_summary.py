"""Summarise ncu reports / launch lists into markdown for profiles/.

    python tools/ncu_summary.py report.ncu-rep [...]      # --set full captures
    python tools/ncu_summary.py --launches launches.csv   # gpu__time_duration list
"""

import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %peak"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active", "IMMA inst %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem %peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise(rep):
    hdr, units, rows = raw(rep)
    lines = [f"### {rep}", "", "| kernel | " + " | ".join(m[1] for m in METRICS) + " |",
             "|---|" + "---|" * len(METRICS)]
    for r in rows:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")
        cells = []
        for m, _ in METRICS:
            # section-prefixed names (e.g. "TPC.TriageCompute.<metric>") count too
            i = hdr.index(m) if m in hdr else next((j for j, h in enumerate(hdr) if h.endswith("." + m)), None)
            cells.append(f"{r[i]} {units[i]}".strip() if i is not None else "n/a")
        lines.append(f"| `{name[:70]}` | " + " | ".join(cells) + " |")
    return "\n".join(lines) + "\n"


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = collections.OrderedDict()
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        tot[name] = tot.get(name, 0.0) + float(r[vi].replace(",", ""))
        cnt[name] += 1
    s = sum(tot.values())
    lines = [f"### launch list {path} ({sum(cnt.values())} launches, cold-cache serialised ncu times)", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k[:70]}` | {cnt[k]} | {v / 1e6:.3f} | {v / s:.3f} |")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--launches":
        for p in args[1:]:
            print(launches(p))
    else:
        for p in args:
            print(summarise(p))
