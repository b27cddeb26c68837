"""Device timeline of graph-replayed generations (CUPTI through
torch.profiler): start / end of every kernel inside the CUDA graph, PDL
overlap included — the in-graph cost of each kernel that per-kernel timing
(cold, serialised) cannot show.

    python scripts/graph_timeline.py [--workload c2] [--gens 4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2501_03944_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--gens", type=int, default=4)
    a = ap.parse_args()
    w = bench.WORKLOADS[a.workload]
    torch.cuda.init()
    eng = P.Engine(bench.make_config(P, w, 1 << 62), P.SearchSpace.box(w["D"], w["lo"], w["hi"]),
                   bench.make_objective(P, w), seed=0)
    eng.initialize()
    eng.enqueue(3)
    eng.sync()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        eng.enqueue(a.gens)
        eng.sync()
    ev = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start:
            ev.append((e.time_range.start, e.time_range.end, e.name))
    ev.sort()
    t0 = ev[0][0] if ev else 0
    rows = [{"k": n[:60], "start_us": round(s - t0, 2), "dur_us": round(e - s, 2)} for s, e, n in ev]
    # per-kernel-name: mean duration and mean "exclusive" span (start -> next start)
    agg = {}
    for i, r in enumerate(rows):
        nxt = rows[i + 1]["start_us"] if i + 1 < len(rows) else r["start_us"] + r["dur_us"]
        d = agg.setdefault(r["k"], {"n": 0, "dur": 0.0, "span": 0.0})
        d["n"] += 1
        d["dur"] += r["dur_us"]
        d["span"] += nxt - r["start_us"]
    total = rows[-1]["start_us"] + rows[-1]["dur_us"] if rows else 0
    print(json.dumps({"workload": a.workload, "gens": a.gens, "total_us": round(total, 1),
                      "per_gen_us": round(total / a.gens, 2),
                      "kernels": {k: {"n": v["n"], "mean_dur_us": round(v["dur"] / v["n"], 2),
                                      "mean_span_us": round(v["span"] / v["n"], 2)} for k, v in agg.items()}},
                     indent=1))
    for r in rows[: 40]:
        print(r)


if __name__ == "__main__":
    main()
