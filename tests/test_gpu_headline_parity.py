"""Parity of the REAL generation path at BASELINE.json's headline shapes.

Every other operator test runs the per-operator seams at D <= 257 (one
512-coordinate chunk).  Here the engine itself runs — the captured CUDA
graph, the objective's own explode variant (bf16 shadow for the tensor-core
objectives), multi-chunk staging of the box and population range — at
D = 25,450 (C2), 61,706 (C3), 100,000 (C4) and 203,530 (C5), and every
step of a generation is checked against the COMPILED REFERENCE
(oracle/_ref: /root/reference/proj/src/engine.cpp, unmodified) fed with the
engine's own inputs:

  initialize           engine.cpp:45-76     positions exact (fp32 image), fitness at tolerance
  explode + mapping    engine.cpp:78-131    sparks exact (fp32 image of the fp64 values)
  bf16 spark shadow    (tensor-core input)  == round-to-nearest-even bf16 of the fp32 sparks
  spark fitness        backend.cpp:15-67    analytic rel 1e-5; NN at the bf16 tolerance
  guiding + guides     engine.cpp:133-196   guides exact (fp32 image), from the engine's fitness
  select + amplitudes  engine.cpp:198-256   bit-exact given the engine's fitness
  loser-out            engine.cpp:258-311   exact decisions / positions / amplitudes / counters
  run loop bookkeeping engine.cpp:386-417   evaluations_used, losers, iterations

Two generations per shape (the second starts from the engine's own state
after the first, with adapted amplitudes and reinitialised losers).  Then
the end-to-end gate: final best over 10 seeds at a fixed evaluation budget
against the compiled reference's finals (tests/golden/finals.npz, made by
tests/golden/make_finals.py), two-sided Mann-Whitney U at alpha = 0.05.

Tolerances (north_star): positional operators exact against
float32(reference) (a 1-ulp clamp where rounding would leave a box whose
bound is not fp32-representable); analytic fitness rel 1e-5; tensor-core
fitness rel 2e-2 + 5e-3 abs against fp64 on the unrounded weights, and
rel 1e-3 + 1e-3 abs (MLP: fp32 accumulation only) / 1e-2 + 2e-3 abs (LeNet:
bf16 activations too) against fp64 on the bf16-rounded weights.
"""
import os

import numpy as np
import pytest

import oracle as O
from tests.impls import f32

pytestmark = pytest.mark.gpu

REL_F32 = 1e-5
REL_BF16, ABS_BF16 = 2e-2, 5e-3
REL_MLP_BF16IN, ABS_MLP_BF16IN = 1e-3, 1e-3
REL_LENET_BF16IN, ABS_LENET_BF16IN = 1e-2, 2e-3
ALPHA = 0.05
WORKERS = os.cpu_count() or 1

# name: (objective descriptor, D, box, mu, lambda, note)
SHAPES = {
    "c2_mlp": (dict(kind=O.OBJ_MLP_WEIGHTS, in_dim=784, hidden=32, out_dim=10, samples=1024), 25450,
               (-1.0, 1.0), 5, 300),
    "c3_lenet": (dict(kind=O.OBJ_LENET, samples=1024), 61706, (-1.0, 1.0), 5, 100),   # lambda 300 -> 100
    "c4_rastrigin": (dict(kind=O.OBJ_RASTRIGIN), 100000, (-5.12, 5.12), 5, 30),
    "c4_ackley": (dict(kind=O.OBJ_ACKLEY), 100000, (-32.768, 32.768), 5, 30),
    "c5_mlp": (dict(kind=O.OBJ_MLP_WEIGHTS, in_dim=784, hidden=256, out_dim=10, samples=1024), 203530,
               (-1.0, 1.0), 4, 64),  # one candidate's shape; population 64 x 1024 -> 4 x 64
}


@pytest.fixture(scope="module")
def P():
    import paper_2501_03944_b200 as P

    return P


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(O.REF_SO):
        pytest.fail(f"{O.REF_SO} missing: build it with `make -C oracle ref` where /root/reference exists")
    return O.Reference()


def _gpu_obj(P, od):
    k = od["kind"]
    if k == O.OBJ_MLP_WEIGHTS:
        return P.MlpWeights(od["in_dim"], od["hidden"], od["out_dim"], od["samples"], 1)
    if k == O.OBJ_LENET:
        return P.LeNet(od["samples"], 1)
    return {O.OBJ_SPHERE: P.Sphere(), O.OBJ_RASTRIGIN: P.Rastrigin(), O.OBJ_ACKLEY: P.Ackley()}[k]


def _box_adjusted(want, lower, upper):
    """fp32 image of the reference; where rounding would leave the box the
    engine keeps the nearest in-box float (1-ulp clamp)."""
    lo32 = np.where(f32(lower) < lower, np.nextafter(f32(lower).astype(np.float32), np.float32(np.inf)),
                    f32(lower).astype(np.float32)).astype(np.float64)
    hi32 = np.where(f32(upper) > upper, np.nextafter(f32(upper).astype(np.float32), np.float32(-np.inf)),
                    f32(upper).astype(np.float32)).astype(np.float64)
    return np.clip(f32(want), lo32, hi32)


def _bf16_bits(x):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


def _bf16_image(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def _check_fitness(ref, od, rows, got, nn_sample):
    """Engine fitness of `rows` (fp32 images) against the reference."""
    desc = O.ObjectiveDesc(**od)
    kind = od["kind"]
    if kind in (O.OBJ_MLP_WEIGHTS, O.OBJ_LENET):
        idx = np.unique(np.linspace(0, rows.shape[0] - 1, nn_sample).astype(int))
        want, _ = ref.batched_apply(desc, rows[idx][None], workers=WORKERS)
        want_b, _ = ref.batched_apply(desc, _bf16_image(rows[idx])[None], workers=WORKERS)
        g = got[idx]
        np.testing.assert_allclose(g, want[0], rtol=REL_BF16, atol=ABS_BF16)
        rel, ab = ((REL_MLP_BF16IN, ABS_MLP_BF16IN) if kind == O.OBJ_MLP_WEIGHTS
                   else (REL_LENET_BF16IN, ABS_LENET_BF16IN))
        np.testing.assert_allclose(g, want_b[0], rtol=rel, atol=ab)
    else:
        want, _ = ref.batched_apply(desc, rows[None], workers=WORKERS)
        np.testing.assert_allclose(got, want[0], rtol=REL_F32, atol=1e-9 * rows.shape[1])


@pytest.mark.parametrize("amp", ["default", "small"])
@pytest.mark.parametrize("name", list(SHAPES))
def test_generation_steps_match_reference_at_headline_shape(P, ref, name, amp):
    """amp = default (A_0 = half the range): a third or more of the spark
    coordinates leave the box, so random mapping is heavily exercised.
    amp = small (A_0 = 1e-5 of the range): improvements are small against the
    spread of the random initial fireworks, so loser-out reinitialises."""
    od, D, (lo, hi), mu, lam = SHAPES[name]
    nn = od["kind"] in (O.OBJ_MLP_WEIGHTS, O.OBJ_LENET)
    B, M, seed = 1, 3, 7
    # a budget of a few waves: iterations_remaining is small (engine.cpp:394-401), so fireworks whose
    # projected improvement cannot reach the batch best become losers (engine.cpp:275-281)
    budget = B * mu + 4 * B * mu * (lam + M)
    lower, upper = np.full(D, lo), np.full(D, hi)
    lower[1::7] = lo / 2  # per-dimension bounds (not a uniform box)
    kw = dict(batches=B, fireworks=mu, sparks_per_firework=lam, guides_per_firework=M,
              boosts=[1.0, 2.0, 4.0], max_evaluations=budget,
              initial_amplitude=0.0 if amp == "default" else 1e-5 * (hi - lo))
    cfg, ocfg = P.MgfwaConfig(**kw), O.Config(**kw)
    desc = O.ObjectiveDesc(**od)
    eng = P.Engine(cfg, P.SearchSpace(lower, upper), _gpu_obj(P, od), seed)
    try:
        # ---- initialize (engine.cpp:45-76)
        eng.initialize()
        st = eng.state()
        rpos, rfit, ramp = ref.initialize(ocfg, lower, upper, desc, seed, workers=WORKERS)
        assert np.array_equal(st.positions, _box_adjusted(rpos, lower, upper))
        assert np.array_equal(st.amplitudes, ramp)
        _check_fitness(ref, od, st.positions.reshape(-1, D), st.fitness.reshape(-1), mu)
        losers_total = 0
        wave = ocfg.evaluations_per_wave()
        max_range = float(np.max(upper - lower))
        for it in (1, 2):
            pre = eng.state()
            assert eng.step(1) == 1
            sp, sf, gd, gf, sh = eng.candidates(bf16=nn)
            # ---- explode + random_mapping(kMapping) (engine.cpp:78-131)
            raw = ref.explode(pre.positions, pre.amplitudes, ocfg, it, seed)
            want = ref.random_mapping(raw, lam, pre.positions, lower, upper, it, seed, O.K_MAPPING)[0]
            bad = np.argwhere(sp != _box_adjusted(want, lower, upper))
            assert bad.size == 0, (name, it, bad[:5])
            oob = np.mean(want != raw[0])
            del raw
            if amp == "default":
                assert oob > 0.01, f"{name}: mapping path barely exercised ({oob:.3%} remapped)"
            if nn:
                assert np.array_equal(sh, _bf16_bits(sp))
            # ---- spark fitness (backend.cpp:15-67)
            _check_fitness(ref, od, sp, sf, 8)
            # ---- guiding vector + guides + random_mapping(kGuide) (engine.cpp:133-196), on the
            #      engine's own spark fitness
            delta = ref.guiding_vector(sp[None], sf[None], ocfg)
            gwant = ref.random_mapping(ref.multi_guiding_sparks(pre.positions, delta, ocfg), M, pre.positions,
                                       lower, upper, it, seed, O.K_GUIDE)[0]
            assert np.array_equal(gd, _box_adjusted(gwant, lower, upper)), (name, it)
            _check_fitness(ref, od, gd, gf, 4)
            # ---- select_best + update_amplitudes (engine.cpp:198-256)
            npos, nfit, nli, imp = ref.select_best(pre.positions, pre.fitness, sp[None], sf[None], lam,
                                                   gd[None], gf[None], M)
            namp = ref.update_amplitudes(pre.amplitudes, imp, ocfg, max_range)
            # ---- loser_out (engine.cpp:258-311) with iterations_remaining of engine.cpp:394-401
            used = pre.evaluations_used + wave
            iters_rem = float(budget - used) / float(wave)
            lpos, lfit, lamp, lli, nl, used_after = ref.loser_out(npos, nfit, namp, nli, used, ocfg, lower, upper,
                                                                  it, seed, iters_rem, desc, workers=WORKERS)
            post = eng.state()
            assert np.array_equal(post.positions, _box_adjusted(lpos, lower, upper)), (name, it)
            assert np.array_equal(post.amplitudes, lamp) and np.array_equal(post.last_improvement, lli)
            moved = np.any(lpos != npos, axis=2)
            assert np.array_equal(post.fitness[~moved], lfit[~moved])
            if moved.any():
                _check_fitness(ref, od, post.positions[moved], post.fitness[moved], mu)
            c = eng.counters()
            losers_total += nl
            assert c["evaluations_used"] == used_after and c["losers_reinitialized"] == losers_total
            assert c["iterations"] == it
        if amp == "small":
            assert losers_total > 0, f"{name}: loser-out path not exercised"
    finally:
        eng.close()


def test_general_draw_path_matches_reference():
    """The explode kernel draws through the chunk-constant form (chunk_draw)
    unless a (key, 512-coordinate chunk) lies within 512 of a carry into the
    mixer's high word (probability 2^-23), which then takes the general form
    (mix_draw).  MGFWA_EXPLODE_GENERAL=1 forces the general form everywhere;
    the headline-shape checks (C2 MLP with the bf16 shadow, C4 Rastrigin with
    the fused fitness, both with heavy random mapping) must stay exact."""
    import subprocess
    import sys

    env = dict(os.environ, MGFWA_EXPLODE_GENERAL="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                          "tests/test_gpu_headline_parity.py", "-k",
                          "generation_steps and default and (c2_mlp or c4_rastrigin)"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "2 passed" in out.stdout, out.stdout[-3000:] + out.stderr[-2000:]


# ------------------------------------------------ 10-seed final best (north_star)
FINALS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "finals.npz")


def _finals_specs():
    import importlib.util

    spec = importlib.util.spec_from_file_location("make_finals", os.path.join(os.path.dirname(FINALS),
                                                                              "make_finals.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.mark.parametrize("name", ["c2_mlp", "c4_rastrigin", "c4_ackley", "c3_lenet_s64", "c5_mlp_reduced"])
def test_final_best_matches_reference_finals(P, name):
    g = np.load(FINALS)
    if f"{name}__finals" not in g.files:
        pytest.fail(f"{name}: no reference finals in {FINALS} (run tests/golden/make_finals.py)")
    m = _finals_specs()
    od, D, (lo, hi), B, mu, lam, M, gens = m.SPECS[name]
    budget = int(g[f"{name}__max_evaluations"])
    assert budget == m.budget(B, mu, lam, M, gens)
    cfg = P.MgfwaConfig(batches=B, fireworks=mu, sparks_per_firework=lam, guides_per_firework=M,
                        boosts=[1.0, 2.0, 4.0][:M], max_evaluations=budget)
    obj = _gpu_obj(P, od)
    finals = []
    for s in g[f"{name}__seeds"]:
        r = P.run(cfg, P.SearchSpace.box(D, lo, hi), obj, int(s))
        assert r.evaluations_used >= budget and np.all(np.diff(r.trace_best, axis=1) <= 0)
        finals.append(r.best_fitness[0])
    from scipy.stats import mannwhitneyu

    cpu = g[f"{name}__finals"]
    p = mannwhitneyu(finals, cpu, alternative="two-sided").pvalue
    print(f"{name}: gpu median {np.median(finals):.6g} reference median {np.median(cpu):.6g} MWU p={p:.3f}")
    assert p > ALPHA, (name, finals, list(cpu), p)
