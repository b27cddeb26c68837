"""Generate the golden fixtures in tests/golden/ from the COMPILED REFERENCE.

Run in the build container (needs /root/reference to build oracle/_ref):

    make -C oracle ref && python tests/golden/make_golden.py

Every array here is produced by the reference's own code
(/root/reference/proj/src/{engine,backend,config,nets}.cpp through
oracle/ref_shim.cpp), except the objective values of the restated objectives
(Rastrigin/Ackley/MLP-weights/LeNet), which come from the shim's C++
restatement plugged in through the reference Objective boundary.  The
fixtures are small (.npz) and travel with the repo; nothing at test time
reads /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def rng_vectors(ref: O.Reference):
    keys = []
    # test_rng.cpp keys plus a sweep over every field
    keys += [(42, 2, 7, 1, 2, 3, 4), (123456789, 1, 0, 5, 6, 7, 8), (11, 4, 3, 4, 5, 6, 7),
             (5, 3, 2, 1, 1, 1, 1), (5, 4, 2, 1, 1, 1, 1), (0, 1, 0, 0, 0, 0, 0),
             (2**64 - 1, 5, 2**40, 7, 63, 1023, 203529)]
    g = np.random.default_rng(7)
    for _ in range(500):
        keys.append((int(g.integers(0, 2**63)), int(g.integers(1, 8)), int(g.integers(0, 10**6)),
                     int(g.integers(0, 8)), int(g.integers(0, 64)), int(g.integers(0, 1024)),
                     int(g.integers(0, 300000))))
    keys = np.array(keys, dtype=np.uint64)
    hashes = np.array([ref.key_hash(*map(int, k)) for k in keys], dtype=np.uint64)
    lo = g.uniform(-10, 0, len(keys))
    hi = lo + g.uniform(0, 20, len(keys))
    hi[:5] = lo[:5]  # degenerate intervals return lo (test_rng.cpp:11-14)
    samples = np.array([ref.uniform_sample(*map(int, k), float(a), float(b))
                        for k, a, b in zip(keys, lo, hi)])
    np.savez_compressed(os.path.join(OUT, "rng.npz"), keys=keys, hashes=hashes, lo=lo, hi=hi,
                        samples=samples)


def operator_vectors(ref: O.Reference):
    """Random-state cases for explode / mapping / guiding / guides / select /
    amplitudes / loser-out, one per seed, on injected inputs."""
    cases = {}
    for case, (B, mu, lam, M, D, sigma) in enumerate([(1, 5, 30, 3, 30, 0.2), (2, 3, 6, 2, 7, 0.34),
                                                      (1, 4, 40, 3, 257, 0.2), (3, 2, 10, 1, 64, 0.5),
                                                      (1, 5, 300, 3, 33, 0.2)]):
        seed = 1000 + case
        g = np.random.default_rng(seed)
        cfg = O.Config(batches=B, fireworks=mu, sparks_per_firework=lam, guides_per_firework=M,
                       guide_fraction=sigma, boosts=[1.0 * 2**m for m in range(M)], max_evaluations=10**6)
        lower = np.full(D, -5.0)
        upper = np.full(D, 5.0)
        lower[::3] = -2.5  # per-dimension bounds
        # fp32-representable state so that a float32 engine sees the same inputs
        pos = g.uniform(lower, upper, size=(B, mu, D)).astype(np.float32).astype(np.float64)
        amp = g.uniform(0.05, 4.0, size=(B, mu)).astype(np.float32).astype(np.float64)
        amp[0, 0] = 0.0
        it = int(g.integers(1, 500))
        sparks = ref.explode(pos, amp, cfg, it, seed)
        mapped = ref.random_mapping(sparks, lam, pos, lower, upper, it, seed, O.K_MAPPING)
        mapped32 = mapped.astype(np.float32).astype(np.float64)
        sfit = (mapped32 ** 2).sum(-1)
        sfit_tie = np.round(sfit, 0)  # forces fitness ties for the stable ranking
        delta = ref.guiding_vector(mapped32, sfit_tie, cfg)
        guides = ref.multi_guiding_sparks(pos, delta, cfg)
        gmapped = ref.random_mapping(guides, M, pos, lower, upper, it, seed, O.K_GUIDE)
        gmapped32 = gmapped.astype(np.float32).astype(np.float64)
        gfit = (gmapped32 ** 2).sum(-1)
        fit = (pos ** 2).sum(-1)
        fit.flat[0] = sfit_tie.reshape(B, mu, lam)[0, 0].min()  # ties with the firework
        npos, nfit, nli, imp = ref.select_best(pos, fit, mapped32, sfit_tie, lam, gmapped32, gfit, M)
        max_range = float((upper - lower).max())
        namp = ref.update_amplitudes(amp, imp, cfg, max_range)
        li = g.uniform(0, 3.0, size=(B, mu)).astype(np.float32).astype(np.float64)
        iters_rem = float(g.uniform(0.5, 40))
        sph = O.ObjectiveDesc(kind=O.OBJ_SPHERE)
        lpos, lfit, lamp, lli, nl, used = ref.loser_out(pos, fit, amp, li, 100, cfg, lower, upper, it, seed,
                                                        iters_rem, sph)
        cases[f"c{case}"] = dict(
            B=B, mu=mu, lam=lam, M=M, D=D, sigma=sigma, seed=seed, it=it, boosts=np.array(cfg.boosts),
            lower=lower, upper=upper, pos=pos, amp=amp, sparks=sparks, mapped=mapped, sfit=sfit_tie,
            delta=delta, guides=guides, gmapped=gmapped, gfit=gfit, fit=fit, npos=npos, nfit=nfit, nli=nli,
            improved=imp, namp=namp, max_range=max_range, li=li, iters_rem=iters_rem, lpos=lpos, lfit=lfit,
            lamp=lamp, lli=lli, nlosers=nl, used_after=used)
    flat = {f"{c}__{k}": np.asarray(v) for c, d in cases.items() for k, v in d.items()}
    np.savez_compressed(os.path.join(OUT, "operators.npz"), **flat)


def run_vectors(ref: O.Reference):
    """Full run() traces (sphere / rastrigin / ackley, small configs)."""
    out = {}
    specs = [
        ("small_sphere", O.Config(batches=2, fireworks=3, sparks_per_firework=6, guides_per_firework=2,
                                  guide_fraction=0.34, boosts=[1.0, 2.0], max_evaluations=1000), 4, -10.0, 10.0,
         O.OBJ_SPHERE, 33),
        ("c1_sphere", O.Config(batches=1, fireworks=5, sparks_per_firework=30, max_evaluations=100000), 30, -10.0,
         10.0, O.OBJ_SPHERE, 0),
        ("c1_rastrigin", O.Config(batches=1, fireworks=5, sparks_per_firework=30, max_evaluations=20000), 30, -5.12,
         5.12, O.OBJ_RASTRIGIN, 1),
        ("ackley", O.Config(batches=2, fireworks=5, sparks_per_firework=20, max_evaluations=5000), 12, -32.768,
         32.768, O.OBJ_ACKLEY, 2),
        ("noguide", O.Config(batches=1, fireworks=4, sparks_per_firework=10, guides_per_firework=0, boosts=[],
                             max_evaluations=2000), 3, -4.0, 4.0, O.OBJ_SPHERE, 9),
    ]
    for name, cfg, D, lo, hi, kind, seed in specs:
        lower, upper = np.full(D, lo), np.full(D, hi)
        rec = ref.run(cfg, lower, upper, O.ObjectiveDesc(kind=kind), seed, workers=0)
        out.update({f"{name}__best_fitness": rec.best_fitness, f"{name}__best_position": rec.best_position,
                    f"{name}__trace_evals": rec.trace_evals, f"{name}__trace_best": rec.trace_best,
                    f"{name}__counters": np.array([rec.evaluations_used, rec.iterations,
                                                   rec.losers_reinitialized, rec.nan_evaluations],
                                                  dtype=np.uint64),
                    f"{name}__seed": np.array(seed), f"{name}__D": np.array(D), f"{name}__lo": np.array(lo),
                    f"{name}__hi": np.array(hi), f"{name}__kind": np.array(kind)})
    np.savez_compressed(os.path.join(OUT, "runs.npz"), **out)


def objective_vectors(ref: O.Reference):
    """Objective values from the reference Objective boundary (shim
    restatements for the new objectives)."""
    g = np.random.default_rng(11)
    out = {}
    for kind, D, scale in [(O.OBJ_SPHERE, 100, 10.0), (O.OBJ_RASTRIGIN, 100, 5.12), (O.OBJ_ACKLEY, 100, 32.0)]:
        X = g.uniform(-scale, scale, size=(6, D)).astype(np.float32).astype(np.float64)
        X[0] = 0.0
        out[f"k{kind}__x"] = X
        out[f"k{kind}__f"] = np.array([ref.evaluate(O.ObjectiveDesc(kind=kind), x) for x in X])
    mlp = O.ObjectiveDesc(kind=O.OBJ_MLP_WEIGHTS, samples=64)
    W = g.uniform(-1, 1, size=(2, mlp.dim())).astype(np.float32).astype(np.float64)
    W[0] = 0.0  # zero weights -> ln(10)
    out["mlp__x"] = W.astype(np.float32)  # exact: fp32-representable
    out["mlp__f"] = np.array([ref.evaluate(mlp, w) for w in W])
    out["mlp__samples"] = np.array(64)
    ln = O.ObjectiveDesc(kind=O.OBJ_LENET, samples=8)
    W = g.uniform(-0.3, 0.3, size=(1, 61706)).astype(np.float32).astype(np.float64)
    out["lenet__x"] = W.astype(np.float32)  # exact: fp32-representable
    out["lenet__f"] = np.array([ref.evaluate(ln, w) for w in W])
    out["lenet__samples"] = np.array(8)
    # reference input-space nets (nets.cpp): net 1 forward on a few inputs
    X = g.uniform(-5, 5, size=(4, 10))
    out["net1__x"] = X
    out["net1__f"] = np.array([ref.evaluate(O.ObjectiveDesc(kind=O.OBJ_NET, net_id=1, weight_seed=1), x) for x in X])
    np.savez_compressed(os.path.join(OUT, "objectives.npz"), **out)


def validation_vectors(ref: O.Reference):
    """Config.validate() messages (config.cpp:42-79) for a set of bad configs."""
    bad = [
        dict(batches=0), dict(amp_amplify=1.0), dict(amp_reduce=1.0), dict(max_evaluations=0),
        dict(guide_fraction=0.6), dict(sparks_per_firework=3, guide_fraction=0.2),
        dict(sparks_per_firework=5, guide_fraction=0.5), dict(boosts=[1.0, 2.0]),
        dict(boosts=[2.0, 2.0, 4.0]), dict(boosts=[1.0, -2.0, 4.0]), dict(),
    ]
    msgs = []
    for kw in bad:
        base = dict(max_evaluations=1000)
        base.update(kw)
        msgs.append(ref.validate(O.Config(**base)) or "")
    import json

    with open(os.path.join(OUT, "validation.json"), "w") as f:
        json.dump({"cases": bad, "messages": msgs}, f, indent=1)


def main():
    O.build(with_reference=True)
    ref = O.Reference()
    rng_vectors(ref)
    operator_vectors(ref)
    run_vectors(ref)
    objective_vectors(ref)
    validation_vectors(ref)
    for fn in sorted(os.listdir(OUT)):
        print(fn, os.path.getsize(os.path.join(OUT, fn)))


if __name__ == "__main__":
    main()
