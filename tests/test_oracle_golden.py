"""Pin the CPU oracle (oracle/mgfwa_oracle.c) against the golden vectors the
compiled reference produced (tests/golden/make_golden.py).  Everything here
must be bit-identical: the oracle is an fp64 restatement with the
reference's arithmetic order."""
import json
import os

import numpy as np
import pytest

import oracle as O
from tests.conftest import GOLDEN, golden_cases


def test_rng_hashes_and_samples(oracle, golden):
    g = golden("rng.npz")
    keys = g["keys"]
    got = np.array([oracle.key_hash(*map(int, k)) for k in keys], dtype=np.uint64)
    assert np.array_equal(got, g["hashes"])
    for k, lo, hi, want in zip(keys, g["lo"], g["hi"], g["samples"]):
        u = oracle.unit_uniform(*map(int, k))
        assert lo + u * (hi - lo) == want


def test_rng_properties(oracle):  # test_rng.cpp:29-83
    vals = [oracle.unit_uniform(9, O.K_MAPPING, i, i % 3, i % 5, i % 7, i % 11) for i in range(10000)]
    assert min(vals) >= 0.0 and max(vals) < 1.0
    s = sum(oracle.unit_uniform(7, O.K_EXPLODE, i // 1000, (i // 100) % 10, (i // 10) % 10, i % 10, i % 7)
            for i in range(200000))
    assert abs(s / 200000 - 0.5) < 0.01
    base = (11, O.K_GUIDE, 3, 4, 5, 6, 7)
    hs = {oracle.key_hash(*base)}
    for delta in range(1, 65):
        for f in (0, 2, 3, 4, 5, 6):
            k = list(base)
            k[f] += delta
            hs.add(oracle.key_hash(*k))
    assert len(hs) == 1 + 64 * 6
    assert oracle.key_hash(5, O.K_MAPPING, 2, 1, 1, 1, 1) != oracle.key_hash(5, O.K_GUIDE, 2, 1, 1, 1, 1)


@pytest.fixture(scope="module")
def cases(golden):
    return golden_cases(golden("operators.npz"))


def test_explode_and_mapping(oracle, cases):
    for name, c in cases.items():
        lam, it, seed = int(c["lam"]), int(c["it"]), int(c["seed"])
        sp = oracle.explode(c["pos"], c["amp"], lam, it, seed)
        assert np.array_equal(sp, c["sparks"]), name
        mp = oracle.random_mapping(sp, lam, c["pos"], c["lower"], c["upper"], it, seed, O.K_MAPPING)
        assert np.array_equal(mp, c["mapped"]), name


def test_guiding_guides_mapping(oracle, cases):
    for name, c in cases.items():
        lam, M = int(c["lam"]), int(c["M"])
        top = int(np.ceil(float(c["sigma"]) * lam))
        d = oracle.guiding_vector(c["mapped"].astype(np.float32).astype(np.float64), c["sfit"], lam, top)
        assert np.array_equal(d, c["delta"]), name
        g = oracle.multi_guiding_sparks(c["pos"], d, c["boosts"])
        assert np.array_equal(g, c["guides"]), name
        gm = oracle.random_mapping(g, M, c["pos"], c["lower"], c["upper"], int(c["it"]), int(c["seed"]), O.K_GUIDE)
        assert np.array_equal(gm, c["gmapped"]), name


def test_select_amplitude_loser(oracle, cases):
    for name, c in cases.items():
        lam, M = int(c["lam"]), int(c["M"])
        m32 = c["mapped"].astype(np.float32).astype(np.float64)
        g32 = c["gmapped"].astype(np.float32).astype(np.float64)
        npos, nfit, nli, imp = oracle.select_best(c["pos"], c["fit"], m32, c["sfit"], lam, g32, c["gfit"], M)
        assert np.array_equal(npos, c["npos"]) and np.array_equal(nfit, c["nfit"]), name
        assert np.array_equal(nli, c["nli"]) and np.array_equal(imp, c["improved"]), name
        amp = oracle.update_amplitudes(c["amp"], imp, 1.2, 0.9, float(c["max_range"]))
        assert np.array_equal(amp, c["namp"]), name
        cfg = O.Config(batches=int(c["B"]), fireworks=int(c["mu"]), sparks_per_firework=lam, guides_per_firework=M,
                       guide_fraction=float(c["sigma"]), boosts=list(c["boosts"]), max_evaluations=10**6)
        p, f, a, l, n = oracle.loser_out(c["pos"], c["fit"], c["amp"], c["li"], cfg, c["lower"], c["upper"],
                                         int(c["it"]), int(c["seed"]), float(c["iters_rem"]),
                                         O.ObjectiveDesc(kind=O.OBJ_SPHERE))
        assert n == int(c["nlosers"]) and 100 + n == int(c["used_after"]), name
        assert np.array_equal(p, c["lpos"]) and np.array_equal(f, c["lfit"]), name
        assert np.array_equal(a, c["lamp"]) and np.array_equal(l, c["lli"]), name


def test_full_runs_bit_identical(oracle, golden):
    g = golden_cases(golden("runs.npz"))
    specs = {
        "small_sphere": O.Config(batches=2, fireworks=3, sparks_per_firework=6, guides_per_firework=2,
                                 guide_fraction=0.34, boosts=[1.0, 2.0], max_evaluations=1000),
        "c1_sphere": O.Config(batches=1, fireworks=5, sparks_per_firework=30, max_evaluations=100000),
        "c1_rastrigin": O.Config(batches=1, fireworks=5, sparks_per_firework=30, max_evaluations=20000),
        "ackley": O.Config(batches=2, fireworks=5, sparks_per_firework=20, max_evaluations=5000),
        "noguide": O.Config(batches=1, fireworks=4, sparks_per_firework=10, guides_per_firework=0, boosts=[],
                            max_evaluations=2000),
    }
    for name, cfg in specs.items():
        c = g[name]
        D = int(c["D"])
        lo, hi = np.full(D, float(c["lo"])), np.full(D, float(c["hi"]))
        r = oracle.run(cfg, lo, hi, O.ObjectiveDesc(kind=int(c["kind"])), int(c["seed"]))
        assert np.array_equal(r.trace_best, c["trace_best"]), name
        assert np.array_equal(r.trace_evals, c["trace_evals"]), name
        assert np.array_equal(r.best_position, c["best_position"]), name
        cnt = c["counters"]
        assert [r.evaluations_used, r.iterations, r.losers_reinitialized, r.nan_evaluations] == list(cnt), name


def test_objectives(oracle, golden):
    g = golden("objectives.npz")
    for kind in (O.OBJ_SPHERE, O.OBJ_RASTRIGIN, O.OBJ_ACKLEY):
        X, F = g[f"k{kind}__x"], g[f"k{kind}__f"]
        for x, f in zip(X, F):
            assert oracle.evaluate(O.ObjectiveDesc(kind=kind), x) == f
    # known answers: Rastrigin(0) = Ackley(0) = 0 (to fp eps), sphere(0) = 0
    assert g["k1__f"][0] == 0.0 and abs(g["k2__f"][0]) < 1e-12 and abs(g["k3__f"][0]) < 1e-12
    mlp = O.ObjectiveDesc(kind=O.OBJ_MLP_WEIGHTS, samples=int(g["mlp__samples"]))
    for x, f in zip(g["mlp__x"].astype(np.float64), g["mlp__f"]):
        assert oracle.evaluate(mlp, x) == f
    assert abs(g["mlp__f"][0] - np.log(10.0)) < 1e-15  # zero weights -> uniform softmax
    ln = O.ObjectiveDesc(kind=O.OBJ_LENET, samples=int(g["lenet__samples"]))
    for x, f in zip(g["lenet__x"].astype(np.float64), g["lenet__f"]):
        assert oracle.evaluate(ln, x) == f


def test_hand_one_sample_mlp(oracle):
    """KAT: a 1-sample MLP whose hidden layer is a single active unit."""
    d = O.ObjectiveDesc(kind=O.OBJ_MLP_WEIGHTS, in_dim=784, hidden=32, out_dim=10, samples=1)
    X, y = oracle.dataset(d)
    w = np.zeros(d.dim())
    # W1[0][0] = 1, b1[0] = 0 -> h0 = x0 ; W2[y][0] = 2 -> z_y = 2 x0 ; others 0
    w[0] = 1.0
    H, I = 32, 784
    w[H * I + H + int(y[0]) * H + 0] = 2.0
    z = np.zeros(10)
    z[int(y[0])] = 2.0 * X[0, 0]
    want = np.log(np.exp(z).sum()) - z[int(y[0])]
    assert abs(oracle.evaluate(d, w) - want) < 1e-15


def test_validation_messages(oracle):
    with open(os.path.join(GOLDEN, "validation.json")) as f:
        v = json.load(f)
    for kw, msg in zip(v["cases"], v["messages"]):
        base = dict(max_evaluations=1000)
        base.update(kw)
        assert (oracle.validate(O.Config(**base)) or "") == msg


def test_dataset_labels_are_balanced(oracle):
    d = O.ObjectiveDesc(kind=O.OBJ_MLP_WEIGHTS, samples=1024)
    X, y = oracle.dataset(d)
    assert X.shape == (1024, 784) and X.min() >= 0.0 and X.max() < 1.0
    assert np.all(X * 256 == np.floor(X * 256))  # 8-bit pixels (exact in bf16)
    counts = np.bincount(y, minlength=10)
    assert counts.min() > 0


@pytest.mark.skipif(not os.path.exists(O.REF_SO), reason="oracle/_ref not built (make -C oracle ref)")
def test_net_objective_checker_is_the_compiled_reference():
    """The paper's benchmark nets are checked against the compiled reference's
    MlpBlackBox (nets.cpp:138-167): the C restatement has no net objective
    (NaN), so smoke() and the GPU tests must use oracle.Reference for them."""
    xs = np.linspace(-3, 3, 10)
    d = O.ObjectiveDesc(kind=O.OBJ_NET, net_id=1, weight_seed=1)
    assert np.isfinite(O.Reference().evaluate(d, xs))
    assert np.isnan(O.Oracle().evaluate(d, xs))
