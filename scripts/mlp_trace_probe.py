"""Runs a few C2 generations (for a %globaltimer-instrumented build's printf)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_03944_b200 as P  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
eng = P.Engine(bench.make_config(P, w, 1 << 62), P.SearchSpace.box(w["D"], w["lo"], w["hi"]),
               bench.make_objective(P, w), seed=0)
eng.initialize()
eng.enqueue(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
eng.sync()
