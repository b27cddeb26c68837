"""Per-kernel device times (CUDA events, back-to-back launches) of one
generation's idempotent kernels on a steady-state C2/C4/C5 engine.

    python scripts/kernel_times.py [--workload c2] [--gens 12] [--iters 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2501_03944_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--gens", type=int, default=12)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    w = bench.WORKLOADS[a.workload]
    eng = P.Engine(bench.make_config(P, w, 1 << 62), P.SearchSpace.box(w["D"], w["lo"], w["hi"]),
                   bench.make_objective(P, w), seed=0)
    eng.initialize()
    eng.enqueue(a.gens)
    eng.sync()
    import time
    t = time.perf_counter()
    eng.enqueue(a.iters)
    eng.sync()
    gen_ms = 1e3 * (time.perf_counter() - t) / a.iters
    out = {"workload": a.workload, "generation_ms_host": gen_ms}
    ks = ["explode", "rank", "guides", "select"] + (["fitness", "guide_fitness"] if w["kind"] in ("mlp", "lenet") else [])
    for k in ks:
        ms, units = eng.time_kernel(k, a.iters)
        out[k + "_us"] = round(1e3 * ms, 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
