"""Expected fraction of explosion coordinates outside the box (the ones that
take the random-mapping path) over a bench-like run: firework positions and
amplitudes from the engine state, Monte-Carlo over U(-1, 1) draws.

    python scripts/oob_rate.py [--workload c2] [--gens 5 50]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_03944_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--gens", type=int, nargs="+", default=[0, 5, 20, 55])
a = ap.parse_args()
w = bench.WORKLOADS[a.workload]
eng = P.Engine(bench.make_config(P, w, 1 << 62), P.SearchSpace.box(w["D"], w["lo"], w["hi"]),
               bench.make_objective(P, w), seed=0)
eng.initialize()
done = 0
rng = np.random.default_rng(0)
for g in a.gens:
    eng.enqueue(g - done)
    eng.sync()
    done = g
    st = eng.state()
    pos, amp = st.positions, st.amplitudes
    fr = []
    for b in range(pos.shape[0]):
        for f in range(pos.shape[1]):
            u = rng.uniform(-1, 1, size=pos.shape[2])
            x = pos[b, f] + amp[b, f] * u
            fr.append(np.mean((x < w["lo"]) | (x > w["hi"])))
    print(f"gen {g}: amplitude median {np.median(amp):.4g}  out-of-box fraction mean {np.mean(fr):.4f}")
