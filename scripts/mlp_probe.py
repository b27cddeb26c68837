"""Probe the tensor-core fitness kernel in isolation (profiling aid).

Times k_mlp_fitness on the C2 spark matrix (1500 candidates) with CUDA
events.  Environment knobs read by the library: MGFWA_MLP_CG=1|2 (CTA
group), MGFWA_MLP_DEBUG_MODE=1 (epilogue releases TMEM without math, i.e.
the TMA + MMA pipeline alone).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2501_03944_b200 as P  # noqa: E402


def main():
    hidden = int(os.environ.get("H", "32"))
    lam = int(os.environ.get("LAM", "300"))
    mu = int(os.environ.get("MU", "5"))
    obj = P.MlpWeights(hidden=hidden)
    cfg = P.MgfwaConfig(batches=1, fireworks=mu, sparks_per_firework=lam, max_evaluations=1 << 62)
    eng = P.Engine(cfg, P.SearchSpace.box(obj.dim(), -1.0, 1.0), obj, seed=0)
    eng.initialize()
    eng.enqueue(1)
    eng.sync()
    ms, units = eng.time_fitness(20)
    flop = 2 * 1024 * (784 * hidden + hidden * 10) * units
    print(json.dumps({"cg": os.environ.get("MGFWA_MLP_CG", "2"), "mode": os.environ.get("MGFWA_MLP_DEBUG_MODE", "0"),
                      "H": hidden, "rows": units, "ms": ms, "tflops": flop / ms / 1e9}))


if __name__ == "__main__":
    main()
