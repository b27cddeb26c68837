"""Firework sharding: a run split over R shards must be
bit-identical to the single-context run — every per-firework operator uses
global (b, n) RNG keys, the exchange replicates exactly the selected state,
and loser-out / record_wave run identically on every shard.

One GPU is available, so R shards are emulated in one process by stepping
them phase by phase (no kernel waits on another) with the in-process
exchange; the NCCL path is exercised with a real 1-rank communicator.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2501_03944_b200 as P

    return P


def _reference(P, cfg, space, obj, seed):
    e = P.Engine(cfg, space, obj, seed)
    e.run()
    r = e.record()
    st = e.state()
    e.close()
    return r, st


def _sharded(P, cfg, space, obj, seed, world):
    shards = [P.Engine(cfg, space, obj, seed, rank=r, world=world) for r in range(world)]
    for s in shards:
        s.initialize()
    wave = cfg.evaluations_per_wave()
    while shards[0].counters()["evaluations_used"] < cfg.max_evaluations:
        for s in shards:
            s.phase(1)
        for dst in shards:
            for src in shards:
                if src is not dst:
                    dst.import_shard(src)
        for s in shards:
            s.phase(2)
        assert wave > 0
    recs = [s.record() for s in shards]
    states = [s.state() for s in shards]
    for s in shards:
        s.close()
    return recs, states


@pytest.mark.parametrize("kind", ["sphere", "rastrigin", "mlp", "lenet", "net"])
@pytest.mark.parametrize("world", [2, 5])
def test_sharded_run_bit_identical(P, kind, world):
    if kind == "mlp":
        obj = P.MlpWeights(samples=128)
        space = P.SearchSpace.box(obj.dim(), -0.5, 0.5)
        budget = 10 + 6 * 2 * 5 * 13
    elif kind == "lenet":
        obj = P.LeNet(samples=64)
        space = P.SearchSpace.box(obj.dim(), -0.3, 0.3)
        budget = 10 + 3 * 2 * 5 * 13
    elif kind == "net":
        obj = P.Net(3, 2)
        space = P.SearchSpace.box(obj.dim(), -5.0, 5.0)
        budget = 10 + 30 * 2 * 5 * 13
    else:
        obj = P.Sphere() if kind == "sphere" else P.Rastrigin()
        space = P.SearchSpace.box(37, -5.12, 5.12)
        budget = 10 + 40 * 2 * 5 * 13
    cfg = P.MgfwaConfig(batches=2, fireworks=5, sparks_per_firework=10, guides_per_firework=3,
                        max_evaluations=budget)
    ref, ref_state = _reference(P, cfg, space, obj, 11)
    recs, states = _sharded(P, cfg, space, obj, 11, world)
    for r, st in zip(recs, states):
        assert np.array_equal(r.trace_best, ref.trace_best)
        assert np.array_equal(r.trace_evaluations, ref.trace_evaluations)
        assert np.array_equal(r.best_position, ref.best_position)
        assert np.array_equal(st.positions, ref_state.positions)
        assert np.array_equal(st.amplitudes, ref_state.amplitudes)
        assert (r.evaluations_used, r.iterations, r.losers_reinitialized) == \
               (ref.evaluations_used, ref.iterations, ref.losers_reinitialized)


@pytest.mark.parametrize("kind", ["sphere", "mlp"])
@pytest.mark.parametrize("mode", ["firework", "replica"])
@pytest.mark.parametrize("graph", ["1", "0"])
def test_nccl_exchange_path_matches(P, kind, mode, graph, monkeypatch):
    """A 1-rank NCCL communicator runs the sharded stepping (phase A, in-place
    all-gather over NCCL, phase B) on one GPU; results must equal the plain
    run bit for bit — with the collectives captured into the generation graph
    and with the fallback of two graphs around host-enqueued collectives
    (MGFWA_NCCL_GRAPH=0, read at capture)."""
    monkeypatch.setenv("MGFWA_NCCL_GRAPH", graph)
    if kind == "mlp":
        obj = P.MlpWeights(samples=128)
        space = P.SearchSpace.box(obj.dim(), -0.5, 0.5)
    else:
        obj = P.Sphere()
        space = P.SearchSpace.box(50, -10.0, 10.0)
    cfg = P.MgfwaConfig(batches=1, fireworks=4, sparks_per_firework=20, max_evaluations=4 + 12 * 4 * 23)
    ref, _ = _reference(P, cfg, space, obj, 5)
    uid = P.Engine.nccl_unique_id()
    assert len(uid) == 128
    e = P.Engine(cfg, space, obj, 5, rank=0, world=1, shard_mode=mode)
    e.attach_nccl(uid)
    e.run()
    r = e.record()
    e.close()
    assert np.array_equal(r.trace_best, ref.trace_best)
    assert np.array_equal(r.best_position, ref.best_position)
    assert r.evaluations_used == ref.evaluations_used


def test_shard_validation(P):
    cfg = P.MgfwaConfig(batches=1, fireworks=5, max_evaluations=1000)
    with pytest.raises(ValueError, match="divisible"):
        P.Engine(cfg, P.SearchSpace.box(4, -1, 1), P.Sphere(), 0, rank=0, world=2)
    cfg2 = P.MgfwaConfig(batches=1, fireworks=4, wall_clock_budget_ms=100.0)
    with pytest.raises(ValueError, match="evaluation budget"):
        P.Engine(cfg2, P.SearchSpace.box(4, -1, 1), P.Sphere(), 0, rank=0, world=2)


def _replica(P, cfg, space, obj, seed, world):
    shards = [P.Engine(cfg, space, obj, seed, rank=r, world=world, shard_mode="replica") for r in range(world)]
    for s in shards:
        s.initialize()
    while shards[0].counters()["evaluations_used"] < cfg.max_evaluations:
        for s in shards:
            s.phase(1)  # ... selection, loser-out of the own batches
        for dst in shards:
            for src in shards:
                if src is not dst:
                    dst.import_shard(src)  # loser counts only
        for s in shards:
            s.phase(2)
    out = [(s.owned_batches, s.record(), s.state(), s.counters()) for s in shards]
    for s in shards:
        s.close()
    return out


@pytest.mark.parametrize("kind", ["sphere", "mlp"])
@pytest.mark.parametrize("batches,world", [(2, 2), (4, 2), (3, 3)])
def test_replica_sharding_matches(P, kind, batches, world):
    """Replica sharding: every rank owns whole
    batches and exchanges only the per-generation loser count; the owned
    batches' traces, best positions and states and the global counters equal
    the single-context run bit for bit."""
    if kind == "mlp":
        obj = P.MlpWeights(samples=128)
        space = P.SearchSpace.box(obj.dim(), -0.5, 0.5)
        budget = batches * (5 + 6 * 5 * 13)
    else:
        obj = P.Sphere()
        space = P.SearchSpace.box(29, -5.12, 5.12)
        budget = batches * (5 + 40 * 5 * 13)
    cfg = P.MgfwaConfig(batches=batches, fireworks=5, sparks_per_firework=10, guides_per_firework=3,
                        max_evaluations=budget)
    ref, ref_state = _reference(P, cfg, space, obj, 5)
    assert ref.losers_reinitialized > 0  # the counter coupling is exercised
    seen = set()
    for owned, r, st, cnt in _replica(P, cfg, space, obj, 5, world):
        seen.update(owned)
        for b in owned:
            assert np.array_equal(r.trace_best[b], ref.trace_best[b])
            assert np.array_equal(r.trace_evaluations[b], ref.trace_evaluations[b])
            assert np.array_equal(r.best_position[b], ref.best_position[b])
            assert np.array_equal(st.positions[b], ref_state.positions[b])
            assert np.array_equal(st.amplitudes[b], ref_state.amplitudes[b])
        for b in set(range(batches)) - set(owned):
            assert np.all(np.isnan(r.trace_best[b][1:]))  # not tracked on this rank
        assert (r.evaluations_used, r.iterations, r.losers_reinitialized) == \
               (ref.evaluations_used, ref.iterations, ref.losers_reinitialized)
    assert seen == set(range(batches))


def test_replica_mode_validation(P):
    cfg = P.MgfwaConfig(batches=3, fireworks=4, max_evaluations=1000)
    space = P.SearchSpace.box(4, -1, 1)
    with pytest.raises(ValueError, match="batches divisible"):
        P.Engine(cfg, space, P.Sphere(), 1, rank=0, world=2, shard_mode="replica")
    with pytest.raises(ValueError, match="shard_mode"):
        P.Engine(cfg, space, P.Sphere(), 1, shard_mode="pipeline")


@pytest.mark.parametrize("mode,world,nccl", [("firework", 2, False), ("firework", 1, True), ("replica", 2, False),
                                             ("replica", 1, True)])
def test_sharded_nan_count_is_global(P, mode, world, nccl):
    """nan_evaluations (backend.cpp:19-22, EvalStats::nan_flagged) of a
    sharded run equals the single-context count: shard-local NaNs (own
    sparks / guides; replica mode: own losers) travel with the exchange and
    are folded once per generation.  Weights of 1e30 overflow the logits to
    inf - inf = NaN, so every evaluation is NaN-flagged."""
    obj = P.MlpWeights(samples=128)
    space = P.SearchSpace.box(obj.dim(), -1e30, 1e30)
    cfg = P.MgfwaConfig(batches=2, fireworks=4, sparks_per_firework=10, guides_per_firework=3,
                        max_evaluations=8 + 5 * 2 * 4 * 13)
    ref, _ = _reference(P, cfg, space, obj, 3)
    assert ref.nan_evaluations > 0
    if nccl:
        e = P.Engine(cfg, space, obj, 3, rank=0, world=1, shard_mode=mode)
        e.attach_nccl(P.Engine.nccl_unique_id())
        e.run()
        r = e.record()
        e.close()
        assert r.nan_evaluations == ref.nan_evaluations
        return
    if mode == "replica":
        outs = _replica(P, cfg, space, obj, 3, world)
        for _, r, _, _ in outs:
            assert r.nan_evaluations == ref.nan_evaluations
    else:
        recs, _ = _sharded(P, cfg, space, obj, 3, world)
        for r in recs:
            assert r.nan_evaluations == ref.nan_evaluations
