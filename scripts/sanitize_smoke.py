"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py

MLP-weights fitness (tcgen05, wide and narrow tiles, SM pairs), LeNet-5
(tcgen05 conv1 + warp-MMA conv2, tcgen05 fc), analytic objectives through the small-problem
cluster loop and through the general graph path, the paper's Net 1, and an
emulated 2-shard firework-sharded run."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_03944_b200 as P  # noqa: E402


def cfg(mu, lam, gens, M=3):
    return P.MgfwaConfig(batches=1, fireworks=mu, sparks_per_firework=lam, guides_per_firework=M,
                         guide_fraction=0.2, boosts=[1.0, 2.0, 4.0][:M], max_evaluations=mu + gens * mu * (lam + M))


def main():
    rng = np.random.default_rng(0)
    for H in (32, 256):
        obj = P.MlpWeights(hidden=H, samples=256)
        W = rng.uniform(-0.05, 0.05, size=(19, obj.dim())).astype(np.float32).astype(np.float64)
        print("mlp", H, P.batched_apply(obj, W)[0][:3])
    r = P.run(cfg(3, 16, 2), P.SearchSpace.box(P.MlpWeights(samples=128).dim(), -1, 1), P.MlpWeights(samples=128), 1)
    print("mlp run", r.best_fitness)
    lo = P.LeNet(samples=200)  # tcgen05 conv1: 3 candidate groups (the last partial), a partial sample chunk
    L = rng.uniform(-0.1, 0.1, size=(29, lo.dim())).astype(np.float32).astype(np.float64)
    print("lenet", P.batched_apply(lo, L)[0][:3])
    print("sphere small", P.run(cfg(5, 30, 3), P.SearchSpace.box(30, -10, 10), P.Sphere(), 2).best_fitness)
    print("rastrigin D=2000", P.run(cfg(5, 30, 2), P.SearchSpace.box(2000, -5.12, 5.12), P.Rastrigin(), 3).best_fitness)
    print("net1", P.run(P.MgfwaConfig(batches=2, fireworks=3, sparks_per_firework=8, max_evaluations=200),
                        P.SearchSpace.box(10, -5, 5), P.Net(1, 1), 4).best_fitness)
    print("ok")


if __name__ == "__main__":
    main()
