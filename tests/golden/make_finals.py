"""Generate tests/golden/finals.npz: final best fitness of the COMPILED
REFERENCE run() (oracle/_ref = /root/reference/proj/src/engine.cpp:313-423)
over 10 seeds at the BASELINE.json headline shapes, each at a fixed
evaluation budget.  tests/test_gpu_headline_parity.py compares the B200
engine's finals on the same configs and seeds against these with a
two-sided Mann-Whitney U test (alpha = 0.05), the north_star's "final best
loss at a fixed evaluation budget statistically indistinguishable from the
reference over 10 seeds".

Run in the build container (needs /root/reference to build oracle/_ref):

    make -C oracle ref && python tests/golden/make_finals.py [name ...]

CPU cost on 8 cores: C2 ~20 min, C4 ~5 min per objective, C3 (S = 64) ~8 min.
Reduced shapes are stated per entry (C3: S = 64 samples; C5: mu = 8,
lambda = 32, S = 128 instead of 64 x 1024 x 1024, which would take days).
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "finals.npz")
SEEDS = list(range(10))

# name: (objective, D, box, B, mu, lambda, M, generations)
SPECS = {
    # BASELINE configs[1]: MLP 784-32-10, S = 1024 (the headline shape, unreduced)
    "c2_mlp": (dict(kind=O.OBJ_MLP_WEIGHTS, in_dim=784, hidden=32, out_dim=10, samples=1024), 25450,
               (-1.0, 1.0), 1, 5, 300, 3, 20),
    # BASELINE configs[3]: D = 1e5 Rastrigin and Ackley (unreduced)
    "c4_rastrigin": (dict(kind=O.OBJ_RASTRIGIN), 100000, (-5.12, 5.12), 1, 5, 30, 3, 50),
    "c4_ackley": (dict(kind=O.OBJ_ACKLEY), 100000, (-32.768, 32.768), 1, 5, 30, 3, 50),
    # BASELINE configs[2]: LeNet-5, D = 61,706, mu = 5, lambda = 300; S reduced 1024 -> 64
    "c3_lenet_s64": (dict(kind=O.OBJ_LENET, samples=64), 61706, (-1.0, 1.0), 1, 5, 300, 3, 8),
    # BASELINE configs[4] shape of one candidate (784-256-10, D = 203,530); population reduced
    "c5_mlp_reduced": (dict(kind=O.OBJ_MLP_WEIGHTS, in_dim=784, hidden=256, out_dim=10, samples=128), 203530,
                       (-1.0, 1.0), 1, 8, 32, 3, 10),
}


def budget(B, mu, lam, M, gens):
    return B * mu + gens * B * mu * (lam + M)


def main(names):
    O.build(with_reference=True)
    ref = O.Reference()
    out = dict(np.load(OUT)) if os.path.exists(OUT) else {}
    workers = os.cpu_count() or 1
    for name in names:
        od, D, (lo, hi), B, mu, lam, M, gens = SPECS[name]
        desc = O.ObjectiveDesc(**od)
        cfg = O.Config(batches=B, fireworks=mu, sparks_per_firework=lam, guides_per_firework=M,
                       boosts=[1.0, 2.0, 4.0][:M], max_evaluations=budget(B, mu, lam, M, gens))
        finals, iters = [], []
        t0 = time.time()
        for s in SEEDS:
            rec = ref.run(cfg, np.full(D, lo), np.full(D, hi), desc, s, workers=workers)
            finals.append(rec.best_fitness[0])
            iters.append(rec.iterations)
            print(f"{name} seed {s}: best {rec.best_fitness[0]:.6g} iters {rec.iterations} "
                  f"({time.time() - t0:.0f} s)", flush=True)
        out[f"{name}__finals"] = np.array(finals)
        out[f"{name}__iterations"] = np.array(iters)
        out[f"{name}__seeds"] = np.array(SEEDS)
        out[f"{name}__max_evaluations"] = np.array(cfg.max_evaluations)
        np.savez_compressed(OUT, **out)


if __name__ == "__main__":
    main(sys.argv[1:] or list(SPECS))
