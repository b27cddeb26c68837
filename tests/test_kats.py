"""The reference's own known-answer tests, re-hosted.

Each test cites the reference test it restates
(/root/reference/proj/tests/test_engine.cpp, test_core.cpp, test_rng.cpp)
and runs against both the CPU oracle (``oracle``, must be bit-identical to
the reference) and the B200 engine (``gpu``, fp32 positions: equalities
hold on the fp32 image of the reference's values).
"""
import numpy as np
import pytest

import oracle as O
from tests.impls import GpuImpl, OracleImpl, f32

IMPLS = [pytest.param("oracle", id="oracle"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]


@pytest.fixture(params=IMPLS)
def impl(request):
    return OracleImpl() if request.param == "oracle" else GpuImpl()


def small_config(**kw):  # test_engine.cpp:16-26
    base = dict(batches=2, fireworks=3, sparks_per_firework=6, guides_per_firework=2, guide_fraction=0.34,
                boosts=[1.0, 2.0], max_evaluations=1000)
    base.update(kw)
    return O.Config(**base)


def box(d, lo, hi):
    return np.full(d, float(lo)), np.full(d, float(hi))


# ---------------------------------------------------------------- initialize
def test_initialize_near_degenerate_box(impl):  # test_engine.cpp:59-69
    c, eps = 1.25, 1e-9
    pos, _, _ = impl.initialize(small_config(), *box(4, c, c + eps), 3)
    assert np.all(pos >= c) and np.all(pos <= c + eps)


def test_initialize_deterministic_per_seed(impl):  # test_engine.cpp:71-80
    lo, hi = box(4, -10, 10)
    a = impl.initialize(small_config(), lo, hi, 7)
    b = impl.initialize(small_config(), lo, hi, 7)
    c = impl.initialize(small_config(), lo, hi, 8)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert not np.array_equal(a[0], c[0])


def test_initial_sphere_fitness_bound(impl):  # test_engine.cpp:82-93
    cfg = small_config(batches=1, fireworks=5)
    pos, fit, _ = impl.initialize(cfg, *box(10, -10, 10), 11)
    assert fit.size == 5
    assert np.all(fit >= 0.0) and np.all(fit <= 1000.0)


# ------------------------------------------------------------------ explode
def test_zero_amplitude_copies_firework(impl):  # test_engine.cpp:95-110
    pos = np.array([1.0, 2.0, -3.0, 4.0]).reshape(1, 2, 2)
    sparks = impl.explode(pos, np.zeros((1, 2)), 4, 1, 99)
    for n in range(2):
        for k in range(4):
            assert np.array_equal(sparks[0, n * 4 + k], pos[0, n])


def test_sparks_inside_amplitude_box(impl):  # test_engine.cpp:112-124
    pos = np.array([5.0]).reshape(1, 1, 1)
    for it in range(1, 201):
        v = impl.explode(pos, np.full((1, 1), 2.0), 1, it, 5)[0, 0, 0]
        assert 3.0 <= v <= 7.0


def test_spark_sample_mean(impl):  # test_engine.cpp:126-142
    pos = np.array([-2.0, 4.0]).reshape(1, 1, 2)
    sparks = impl.explode(pos, np.full((1, 1), 3.0), 100000, 1, 17)
    mean = sparks[0].mean(axis=0)
    assert np.all(np.abs(mean - pos[0, 0]) < 0.02 * 3.0)


# ------------------------------------------------------------------ mapping
def test_mapping_leaves_in_bounds_untouched(impl):  # test_engine.cpp:144-156
    pos = np.array([0, 1, 2, -1, -2, -3, 3, 2, 1, 0, 0, 0, 1, 1, 1, 2, 2, 2], float).reshape(2, 3, 3)
    cand = np.full((2, 6, 3), 0.5)
    out = impl.random_mapping(cand, 2, pos, *box(3, -5, 5), 1, 5, O.K_MAPPING)
    assert np.array_equal(out, cand)


def test_collapsed_population_maps_to_point(impl):  # test_engine.cpp:158-176
    pos = np.array([1.5, -0.5]).reshape(1, 1, 2)
    cand = np.array([9.0, 1.0, -8.0, 2.0, 7.0, -6.0]).reshape(1, 3, 2)
    out = impl.random_mapping(cand, 3, pos, *box(2, -5, 5), 2, 5, O.K_MAPPING)
    assert out[0, 0, 0] == 1.5 and out[0, 0, 1] == 1.0
    assert out[0, 1, 0] == 1.5 and out[0, 1, 1] == 2.0
    assert out[0, 2, 0] == 1.5 and out[0, 2, 1] == -0.5


def test_mapping_lands_in_population_range(impl):  # test_engine.cpp:178-219
    o = O.Oracle()
    for seed in range(50):
        cfg = small_config()
        dims = 1 + seed % 5
        lo, hi = box(dims, -4, 4)
        pos, _, _ = impl.initialize(cfg, lo, hi, seed)
        wild = np.array([o.unit_uniform(seed, O.K_EXPLODE, 999, i, 0, 0, 0) * 100.0 - 50.0
                         for i in range(2 * 3 * 4 * dims)]).reshape(2, 12, dims)
        if not impl.exact:
            wild = f32(wild)
        out = impl.random_mapping(wild, 4, pos, lo, hi, 3, seed, O.K_MAPPING)
        for b in range(2):
            plo, phi = pos[b].min(axis=0), pos[b].max(axis=0)
            inside = (wild[b] >= -4.0) & (wild[b] <= 4.0)
            assert np.array_equal(out[b][inside], wild[b][inside])
            assert np.all(out[b][~inside] >= np.broadcast_to(plo, wild[b].shape)[~inside])
            assert np.all(out[b][~inside] <= np.broadcast_to(phi, wild[b].shape)[~inside])
            assert np.all(out[b] >= -4.0) and np.all(out[b] <= 4.0)


# ----------------------------------------------------------------- guiding
def test_guiding_one_best_one_worst(impl):  # test_engine.cpp:221-233
    sparks = np.array([1.0, 1.0, 3.0, 3.0]).reshape(1, 2, 2)
    d = impl.guiding_vector(sparks, np.array([[0.0, 10.0]]), 2, 1)
    assert d[0, 0, 0] == -2.0 and d[0, 0, 1] == -2.0


def test_identical_sparks_zero_guide(impl):  # test_engine.cpp:235-246
    sparks = np.full((1, 6, 3), 2.5)
    d = impl.guiding_vector(sparks, np.arange(6.0).reshape(1, 6), 6, 3)
    assert np.all(d == 0.0)


def test_guiding_hand_computed(impl):  # test_engine.cpp:248-267
    sparks = np.arange(1.0, 9.0).reshape(1, 4, 2)
    d = impl.guiding_vector(sparks, np.array([[3.0, 1.0, 7.0, 5.0]]), 4, 2)
    assert d[0, 0, 0] == -4.0 and d[0, 0, 1] == -4.0


def test_ranking_ties_by_index(impl):  # test_engine.cpp:269-279
    sparks = np.array([10.0, 20.0]).reshape(1, 2, 1)
    d = impl.guiding_vector(sparks, np.full((1, 2), 4.0), 2, 1)
    assert d[0, 0, 0] == -10.0


def test_guiding_golden_random(impl, golden):  # engine.cpp:133-172 on reference vectors
    from tests.conftest import golden_cases

    for name, c in golden_cases(golden("operators.npz")).items():
        lam, top = int(c["lam"]), int(np.ceil(float(c["sigma"]) * int(c["lam"])))
        d = impl.guiding_vector(c["mapped"].astype(np.float32).astype(np.float64), c["sfit"], lam, top)
        ref = c["delta"]
        if impl.exact:
            assert np.array_equal(d, ref), name
        else:
            assert np.array_equal(d, f32(ref)), name  # fp64 arithmetic, one rounding


# ------------------------------------------------------------------ guides
def test_zero_delta_collapses_guides(impl):  # test_engine.cpp:281-299
    pos = np.array([1, 2, 3, 4, 5, 6, -1, -2, -3, -4, -5, -6], float).reshape(2, 3, 2)
    g = impl.multi_guiding_sparks(pos, np.zeros((2, 3, 2)), [1.0, 2.0, 4.0])
    for b in range(2):
        for n in range(3):
            for m in range(3):
                assert np.array_equal(g[b, n * 3 + m], pos[b, n])


def test_boosts_scale_linearly(impl):  # test_engine.cpp:301-312
    g = impl.multi_guiding_sparks(np.zeros((1, 1, 2)), np.array([1.0, -1.0]).reshape(1, 1, 2), [1.0, 2.0])
    assert g[0, 0, 0] == 1.0 and g[0, 0, 1] == -1.0 and g[0, 1, 0] == 2.0 and g[0, 1, 1] == -2.0


def test_every_guide_is_pos_plus_boosted(impl):  # test_engine.cpp:314-337
    o = O.Oracle()
    lo, hi = box(3, -5, 5)
    pos, _, _ = impl.initialize(small_config(guides_per_firework=3, boosts=[1.0, 2.0, 4.0]), lo, hi, 21)
    delta = np.array([o.unit_uniform(13, O.K_GUIDE, i, 0, 0, 0, 0) * 4.0 - 2.0 for i in range(18)]).reshape(2, 3, 3)
    if not impl.exact:
        delta = f32(delta)
    g = impl.multi_guiding_sparks(pos, delta, [1.0, 2.0, 4.0])
    for m, beta in enumerate([1.0, 2.0, 4.0]):
        want = pos + beta * delta
        if not impl.exact:
            want = f32(want)
        assert np.array_equal(g[:, m::3, :], want)


# ------------------------------------------------------------------ select
def test_selection_keeps_firework(impl):  # test_engine.cpp:363-374
    npos, nfit, nli, imp = impl.select_best(np.zeros((1, 1, 2)), np.array([[1.0]]),
                                            np.array([1, 1, 2, 2], float).reshape(1, 2, 2),
                                            np.array([[5.0, 9.0]]), 2)
    assert nfit[0, 0] == 1.0 and npos[0, 0, 0] == 0.0 and nli[0, 0] == 0.0 and imp[0, 0] == 0.0


def test_strictly_better_spark_replaces(impl):  # test_engine.cpp:376-387
    npos, nfit, nli, imp = impl.select_best(np.zeros((1, 1, 2)), np.array([[1.0]]),
                                            np.array([1, 1, 2, 2], float).reshape(1, 2, 2),
                                            np.array([[0.25, 9.0]]), 2)
    assert nfit[0, 0] == 0.25 and npos[0, 0, 0] == 1.0 and nli[0, 0] == 0.75 and imp[0, 0] == 1.0


def test_selection_brute_force(impl):  # test_engine.cpp:389-441
    o = O.Oracle()
    B, mu, lam, M, D = 2, 3, 4, 2, 2
    for seed in range(30):
        def fill(count, stream):
            return np.array([o.unit_uniform(seed, stream, i, 1, 0, 0, 0) * 20.0 - 10.0 for i in range(count)])

        pos = fill(B * mu * D, O.K_INIT).reshape(B, mu, D)
        sparks = fill(B * mu * lam * D, O.K_EXPLODE).reshape(B, mu * lam, D)
        guides = fill(B * mu * M * D, O.K_GUIDE).reshape(B, mu * M, D)
        fit = np.array([[o.unit_uniform(seed, O.K_REINIT, 0, b, n, 0, 0) * 10.0 for n in range(mu)]
                        for b in range(B)])
        sfit = np.array([[o.unit_uniform(seed, O.K_REINIT, 1, b, n, k, 0) * 10.0 for n in range(mu)
                          for k in range(lam)] for b in range(B)])
        gfit = np.array([[o.unit_uniform(seed, O.K_REINIT, 2, b, n, m, 0) * 10.0 for n in range(mu)
                          for m in range(M)] for b in range(B)])
        if not impl.exact:  # the engine keeps fitness in fp32
            sfit, gfit = f32(sfit), f32(gfit)
            pos, sparks, guides = f32(pos), f32(sparks), f32(guides)
        npos, nfit, nli, _ = impl.select_best(pos, fit, sparks, sfit, lam, guides, gfit, M)
        for b in range(B):
            for n in range(mu):
                best = min(fit[b, n], sfit[b, n * lam:(n + 1) * lam].min(), gfit[b, n * M:(n + 1) * M].min())
                assert nfit[b, n] == best
                assert nli[b, n] == max(0.0, fit[b, n] - best)


# --------------------------------------------------------------- amplitude
def test_amplitude_rule(impl):  # test_engine.cpp:443-451
    nxt = impl.update_amplitudes(np.ones((1, 2)), np.array([[1.0, 0.0]]), 1.2, 0.9, 20.0)
    assert abs(nxt[0, 0] - 1.2) <= 1.2e-12 and abs(nxt[0, 1] - 0.9) <= 0.9e-12


def test_amplitude_floor(impl):  # test_engine.cpp:453-473
    a = np.ones((1, 1))
    for _ in range(100):
        a = impl.update_amplitudes(a, np.zeros((1, 1)), 1.2, 0.6, 20.0)
        assert a[0, 0] > 0.0
    assert a[0, 0] == 2e-11
    for _ in range(300):
        a = impl.update_amplitudes(a, np.zeros((1, 1)), 1.2, 0.9, 20.0)
        assert a[0, 0] > 0.0
    assert a[0, 0] == 2e-11


def test_amplitude_ceiling(impl):  # test_engine.cpp:475-481
    assert impl.update_amplitudes(np.full((1, 1), 19.0), np.ones((1, 1)), 1.2, 0.9, 20.0)[0, 0] == 20.0


# ---------------------------------------------------------------- loser-out
def _loser_state():
    pos = np.array([0, 0, 1, 1, 2, 2], float).reshape(1, 3, 2)
    fit = np.array([[1.0, 11.0, 11.0]])
    return pos, fit, np.ones((1, 3)), np.zeros((1, 3))


@pytest.mark.parametrize("case", ["rates", "slow", "nohorizon", "catchup"])
def test_loser_out_table(impl, case):  # test_engine.cpp:483-547
    cfg = small_config(batches=1, fireworks=3)
    lo, hi = box(2, -5, 5)
    pos, fit, amp, li = _loser_state()
    iters = 20.0
    if case == "rates":
        li[0] = [5.0, 0.1, 0.0]
    elif case == "slow":
        fit[0, 1] = 2.0
        li[0] = [5.0, 0.1, 0.0]
    elif case == "nohorizon":
        iters = 0.0
    else:
        li[0] = [0.0, 0.0, 10.0]
    p, f, a, l, n, used = impl.loser_out(pos, fit, amp, li, 3, cfg, lo, hi, 1, 42, iters)
    if case == "rates":
        assert n == 2 and p[0, 0, 0] == 0.0 and f[0, 0] == 1.0
        assert p[0, 1, 0] != 1.0 and p[0, 2, 0] != 2.0 and l[0, 1] == 0.0 and used == 5
    elif case == "slow":
        assert n == 1 and p[0, 1, 0] == 1.0 and p[0, 2, 0] != 2.0
    elif case == "nohorizon":
        assert n == 0
    else:
        assert n == 1 and p[0, 2, 0] == 2.0
        assert a[0, 1] == 5.0  # resolved_initial_amplitude(max_range = 10)
        fresh, _ = impl.batched_apply(O.OBJ_SPHERE, p[0, 1:2])
        assert f[0, 1] == fresh[0]


# --------------------------------------------------------------------- run
def test_run_exact_init_budget(impl):  # test_engine.cpp:549-560
    cfg = small_config(max_evaluations=6)
    r = impl.run(cfg, *box(4, -10, 10), O.OBJ_SPHERE, 5)
    assert r.trace_evals.shape == (2, 1)
    assert r.evaluations_used == 6 and r.iterations == 0


def test_run_budget_too_small(impl):  # test_engine.cpp:562-569
    cfg = small_config(max_evaluations=5)
    with pytest.raises(ValueError, match="budget too small"):
        impl.run(cfg, *box(4, -10, 10), O.OBJ_SPHERE, 5)


def test_run_reproducible(impl):  # test_engine.cpp:571-584
    cfg = small_config(max_evaluations=400)
    a = impl.run(cfg, *box(4, -10, 10), O.OBJ_SPHERE, 33)
    b = impl.run(cfg, *box(4, -10, 10), O.OBJ_SPHERE, 33)
    assert np.array_equal(a.trace_best, b.trace_best) and np.array_equal(a.trace_evals, b.trace_evals)
    assert np.array_equal(a.best_position, b.best_position)


def test_run_monotone_in_bounds_coherent(impl):  # test_engine.cpp:586-610
    for seed in range(10):
        cfg = small_config(max_evaluations=600)
        lo, hi = box(3, -4, 4)
        r = impl.run(cfg, lo, hi, O.OBJ_SPHERE, seed)
        assert np.all(np.diff(r.trace_best, axis=1) <= 0)
        assert np.all(np.diff(r.trace_evals.astype(np.int64), axis=1) > 0)
        assert np.all(r.best_position >= -4.0) and np.all(r.best_position <= 4.0)
        fit, _ = impl.batched_apply(O.OBJ_SPHERE, r.best_position)
        assert np.array_equal(r.best_fitness, fit)


def test_run_eval_accounting(impl):  # test_engine.cpp:612-622
    cfg = small_config(max_evaluations=500)
    r = impl.run(cfg, *box(3, -4, 4), O.OBJ_SPHERE, 3)
    wave, slack = cfg.evaluations_per_wave(), cfg.batches * (cfg.fireworks - 1)
    assert 500 <= r.evaluations_used < 500 + wave + slack


def test_run_without_guides_improves(impl):  # test_engine.cpp:624-633
    cfg = small_config(guides_per_firework=0, boosts=[], max_evaluations=2000)
    r = impl.run(cfg, *box(3, -4, 4), O.OBJ_SPHERE, 9)
    assert r.trace_best[0, -1] < r.trace_best[0, 0]


def test_run_strong_progress(impl):  # test_engine.cpp:635-644
    cfg = O.Config(batches=1, fireworks=5, max_evaluations=20000)
    r = impl.run(cfg, *box(5, -10, 10), O.OBJ_SPHERE, 1)
    assert r.trace_best[0, -1] < r.trace_best[0, 0] / 100.0


# --------------------------------------------------------------- backend
def test_argmin_basics(impl):  # test_core.cpp:111-134
    idx, val = impl.argmin(np.array([[5.0, 3.0, 9.0]]))
    assert idx[0] == 1 and val[0] == 3.0
    idx, val = impl.argmin(np.full((1, 3), 2.0))
    assert idx[0] == 0 and val[0] == 2.0
    idx, val = impl.argmin(np.full((1, 4), np.inf))
    assert idx[0] == 0 and np.isinf(val[0])


def test_argmin_exhaustive(impl):  # test_core.cpp:136-159
    o = O.Oracle()
    for seed in range(20):
        f = np.array([[o.unit_uniform(seed, O.K_INIT, 1, b, n, 0, 0) * 200 - 100 for n in range(16)]
                      for b in range(8)])
        idx, val = impl.argmin(f)
        assert np.array_equal(idx, np.argmin(f, axis=1).astype(np.uint64))
        assert np.array_equal(val, f.min(axis=1))


def test_nan_becomes_inf_and_counted(impl):  # test_core.cpp:94-109 (NaN rows)
    rows = np.array([[1.0, 2.0], [np.nan, 0.0], [3.0, np.nan], [0.5, 0.5]])
    fit, nan = impl.batched_apply(O.OBJ_SPHERE, rows)
    assert not np.any(np.isnan(fit))
    assert np.isinf(fit[1]) and np.isinf(fit[2]) and nan == 2


def test_zero_cube_sum(impl):  # test_core.cpp:63-68
    fit, _ = impl.batched_apply(O.OBJ_SPHERE, np.zeros((6, 5)))
    assert np.all(fit == 0.0)
