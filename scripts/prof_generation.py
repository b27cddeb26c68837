"""Profiling driver: a few C2 generations with a fixed kernel order, for
`ncu -k regex:<kernel> -s <skip> -c 1` captures of the hot kernels.

Launch order per generation (graph replay): k_explode_map,
k_mlp_fitness(sparks), k_rank, k_guides, k_mlp_fitness(guides), k_select,
k_loser, k_fresh_rows, k_mlp_fitness(fresh),
k_finalize_record, k_record_copy.  initialize() launches k_fresh_rows,
k_mlp_fitness(fresh), k_finalize_record, k_record_copy first.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2501_03944_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gens", type=int, default=3)
    ap.add_argument("--workload", default="c2")
    a = ap.parse_args()
    if a.workload == "c2":
        obj, D, lo, hi, lam = P.MlpWeights(), 25450, -1.0, 1.0, 300
    elif a.workload == "c4":
        obj, D, lo, hi, lam = P.Rastrigin(), 100000, -5.12, 5.12, 30
    else:
        obj, D, lo, hi, lam = P.Sphere(), 30, -10.0, 10.0, 30
    cfg = P.MgfwaConfig(batches=1, fireworks=5, sparks_per_firework=lam, max_evaluations=1 << 62)
    eng = P.Engine(cfg, P.SearchSpace.box(D, lo, hi), obj, seed=0)
    eng.initialize()
    eng.enqueue(a.gens)
    eng.sync()
    print("ok", eng.counters())


if __name__ == "__main__":
    main()
