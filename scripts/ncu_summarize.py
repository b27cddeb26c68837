"""Summarise ncu captures into profiles/ (text, committed).

    python scripts/ncu_summarize.py launches <launches.csv> <out.md> [first_n_launches]
    python scripts/ncu_summarize.py report <a.ncu-rep> [<b.ncu-rep> ...] <out.json>
"""
import collections
import csv
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__warps_active.avg.per_cycle_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def launches(path, out, first=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.OrderedDict()
    n = collections.Counter()
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    seen = 0
    for r in data:
        if r[mi] != "gpu__time_duration.sum":
            continue
        seen += 1
        if first is not None and seen > first:
            break
        name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        t = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        tot[name] = tot.get(name, 0.0) + t
        n[name] += 1
    total = sum(tot.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary ({path})\n\n")
        if first is not None:
            f.write(f"First {first} launches only (initialize + the bench's generations; the later\n"
                    "roofline timing launches of the fitness kernel are excluded).\n\n")
        f.write("Cold-cache, serialised per-launch times (`--metrics gpu__time_duration.sum "
                "--clock-control none`): compare SHARES, not absolutes.\n\n")
        f.write("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"| {k} | {n[k]} | {v:.1f} | {v / n[k]:.2f} | {100 * v / total:.1f}% |\n")
        f.write(f"\nTotal {total:.1f} us over {sum(n.values())} launches.\n")


def report(paths, out):
    res = []
    for p in paths:
        txt = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(txt.splitlines()))
        h, units, data = rows[0], rows[1], rows[2:]
        for r in data:
            import os
            base = os.path.basename(p)
            d = {"report": p, "kernel": r[h.index("Kernel Name")],
                 "workload": base.split("_")[0] if base[:1] == "c" and "_" in base else "c2"}
            for m in METRICS:
                if m in h:
                    i = h.index(m)
                    d[m] = f"{r[i]} {units[i]}".strip()
            res.append(d)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else None)
    else:
        report(sys.argv[2:-1], sys.argv[-1])
