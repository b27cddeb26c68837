"""Multi-rank firework sharding on CPU (world_size 2, gloo).

The sharded decomposition the B200 engine uses across GPUs (DESIGN.md §5,
SURVEY.md §8(e)) restated on the fp64 oracle: each rank explodes / maps /
evaluates / guides / selects only its own fireworks (global (b, n) RNG keys),
the selected {position, fitness, amplitude, last improvement} are
all-gathered every generation, and loser-out + record_wave run on the
replicated state on every rank.  Both ranks must reproduce the unsharded
run() (engine.cpp:313-423) bit for bit.
"""
import os
import socket

import numpy as np
import pytest

import oracle as O

M64 = (1 << 64) - 1


def _smix(x):
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def _prefix(seed, stream, it, b, n):
    h = _smix(np.uint64(seed))
    for f in (stream, it, b, n):
        h = _smix(h ^ np.uint64(f))
    return h


def _uniform(seed, stream, it, b, n, K, D, lo, hi):
    """uniform_sample over a [K][D] grid of keys (rng.hpp:43-65), vectorised."""
    pre = _prefix(seed, stream, it, b, n)
    k = np.arange(K, dtype=np.uint64)[:, None]
    d = np.arange(D, dtype=np.uint64)[None, :]
    h = _smix(_smix(pre ^ k) ^ d)
    u = (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return lo + u * (hi - lo)


def _map(cand, seed, stream, it, b, n, lower, upper, plo, phi):
    out = cand.copy()
    K, D = cand.shape
    bad = ~((cand >= lower[None, :]) & (cand <= upper[None, :]))
    if bad.any():
        draw = _uniform(seed, stream, it, b, n, K, D, np.broadcast_to(plo, (K, D)), np.broadcast_to(phi, (K, D)))
        out[bad] = draw[bad]
    return out


def _sharded_run(rank, world, cfg, lower, upper, seed, kind):
    import torch
    import torch.distributed as dist

    o = O.Oracle()
    desc = O.ObjectiveDesc(kind=kind)
    B, mu, lam, M = cfg.batches, cfg.fireworks, cfg.sparks_per_firework, cfg.guides_per_firework
    assert B == 1 and mu % world == 0
    D = lower.size
    ml = mu // world
    f_lo = rank * ml
    top = cfg.top_spark_count()
    max_range = float(np.max(upper - lower))
    a0 = cfg.initial_amplitude if cfg.initial_amplitude > 0 else 0.5 * max_range
    wave = cfg.evaluations_per_wave()

    pos = o.initialize_positions(cfg, lower, upper, seed)  # [1][mu][D], all ranks
    fit, _ = o.batched_apply(desc, pos)
    amp = np.full((1, mu), a0)
    li = np.zeros((1, mu))
    used = B * mu
    best = np.array([np.inf])
    best_pos = np.zeros((1, D))
    trace = []

    def record():
        i = int(np.argmin(fit[0]))  # lowest index on ties, like argmin_per_population
        v = fit[0, i]
        for j in range(mu):
            if fit[0, j] < v:
                v, i = fit[0, j], j
        if v < best[0]:
            best[0] = v
            best_pos[0] = pos[0, i]
        trace.append((used, best[0]))

    record()
    it = 0
    while used < cfg.max_evaluations:
        it += 1
        plo, phi = pos[0].min(axis=0), pos[0].max(axis=0)
        # ---- owned fireworks: explode + map + fitness
        sparks = np.empty((1, ml * lam, D))
        for j in range(ml):
            n = f_lo + j
            raw = pos[0, n][None, :] + _uniform(seed, O.K_EXPLODE, it, 0, n, lam, D, -1.0, 1.0) * amp[0, n]
            sparks[0, j * lam:(j + 1) * lam] = _map(raw, seed, O.K_MAPPING, it, 0, n, lower, upper, plo, phi)
        sfit, _ = o.batched_apply(desc, sparks)
        # ---- guiding sparks of the owned fireworks
        lpos = pos[:, f_lo:f_lo + ml]
        if M > 0:
            delta = o.guiding_vector(sparks, sfit, lam, top)
            guides = np.empty((1, ml * M, D))
            for j in range(ml):
                n = f_lo + j
                g = np.stack([lpos[0, j] + cfg.boosts[m] * delta[0, j] for m in range(M)])
                guides[0, j * M:(j + 1) * M] = _map(g, seed, O.K_GUIDE, it, 0, n, lower, upper, plo, phi)
            gfit, _ = o.batched_apply(desc, guides)
            npos, nfit, nli, imp = o.select_best(lpos, fit[:, f_lo:f_lo + ml], sparks, sfit, lam, guides, gfit, M)
        else:
            npos, nfit, nli, imp = o.select_best(lpos, fit[:, f_lo:f_lo + ml], sparks, sfit, lam)
        namp = o.update_amplitudes(amp[:, f_lo:f_lo + ml], imp, cfg.amp_amplify, cfg.amp_reduce, max_range)
        # ---- the per-generation exchange (all-gather of the selected fireworks)
        rec = torch.from_numpy(np.concatenate([npos[0].reshape(-1), nfit[0], namp[0], nli[0]]))
        out = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(out, rec)
        for r, t in enumerate(out):
            a = t.numpy()
            sl = slice(r * ml, (r + 1) * ml)
            pos[0, sl] = a[:ml * D].reshape(ml, D)
            fit[0, sl] = a[ml * D:ml * D + ml]
            amp[0, sl] = a[ml * D + ml:ml * D + 2 * ml]
            li[0, sl] = a[ml * D + 2 * ml:]
        used += wave
        # ---- replicated: loser-out (engine.cpp:258-311) and record_wave
        left = cfg.max_evaluations - used if cfg.max_evaluations > used else 0
        pos, fit, amp, li, nl = o.loser_out(pos, fit, amp, li, cfg, lower, upper, it, seed, left / wave, desc)
        used += nl
        record()
    return np.array(trace), best_pos, used, it


def _replica_run(rank, world, cfg, lower, upper, seed, kind):
    """Replica sharding: rank r owns batch r
    (B == world, one batch each); the only per-generation exchange is the
    loser count, which the shared evaluation budget needs (engine.cpp:309)."""
    import torch
    import torch.distributed as dist

    o = O.Oracle()
    desc = O.ObjectiveDesc(kind=kind)
    B, mu, lam, M = cfg.batches, cfg.fireworks, cfg.sparks_per_firework, cfg.guides_per_firework
    assert B == world
    b = rank
    D = lower.size
    top = cfg.top_spark_count()
    max_range = float(np.max(upper - lower))
    wave = cfg.evaluations_per_wave()

    pos = o.initialize_positions(cfg, lower, upper, seed)  # [B][mu][D]: initialize is global
    fit, _ = o.batched_apply(desc, pos)
    a0 = cfg.initial_amplitude if cfg.initial_amplitude > 0 else 0.5 * max_range
    amp = np.full((B, mu), a0)
    li = np.zeros((B, mu))
    used = B * mu
    best, best_pos, trace = np.inf, np.zeros(D), []

    def record():
        nonlocal best, best_pos
        v, i = fit[b, 0], 0
        for j in range(1, mu):
            if fit[b, j] < v:
                v, i = fit[b, j], j
        if v < best:
            best, best_pos = v, pos[b, i].copy()
        trace.append((used, best))

    record()
    it = 0
    while used < cfg.max_evaluations:
        it += 1
        plo, phi = pos[b].min(axis=0), pos[b].max(axis=0)
        sparks = np.empty((1, mu * lam, D))
        for n in range(mu):
            raw = pos[b, n][None, :] + _uniform(seed, O.K_EXPLODE, it, b, n, lam, D, -1.0, 1.0) * amp[b, n]
            sparks[0, n * lam:(n + 1) * lam] = _map(raw, seed, O.K_MAPPING, it, b, n, lower, upper, plo, phi)
        sfit, _ = o.batched_apply(desc, sparks)
        lpos = pos[b:b + 1]
        delta = o.guiding_vector(sparks, sfit, lam, top)
        guides = np.empty((1, mu * M, D))
        for n in range(mu):
            g = np.stack([lpos[0, n] + cfg.boosts[m] * delta[0, n] for m in range(M)])
            guides[0, n * M:(n + 1) * M] = _map(g, seed, O.K_GUIDE, it, b, n, lower, upper, plo, phi)
        gfit, _ = o.batched_apply(desc, guides)
        npos, nfit, nli, imp = o.select_best(lpos, fit[b:b + 1], sparks, sfit, lam, guides, gfit, M)
        namp = o.update_amplitudes(amp[b:b + 1], imp, cfg.amp_amplify, cfg.amp_reduce, max_range)
        pos[b], fit[b], amp[b], li[b] = npos[0], nfit[0], namp[0], nli[0]
        used += wave
        # loser-out of the own batch: the other batches get equal fitness and
        # zero improvement rates, which never makes a loser
        left = cfg.max_evaluations - used if cfg.max_evaluations > used else 0
        p_, f_, a_, l_ = pos.copy(), np.zeros_like(fit), amp.copy(), np.zeros_like(li)
        f_[b], l_[b] = fit[b], li[b]
        p_, f_, a_, l_, nl = o.loser_out(p_, f_, a_, l_, cfg, lower, upper, it, seed, left / wave, desc)
        pos[b], fit[b], amp[b], li[b] = p_[b], f_[b], a_[b], l_[b]
        t = torch.tensor([nl], dtype=torch.int64)
        dist.all_reduce(t)  # the exchange: losers of every batch
        used += int(t.item())
        record()
    return np.array(trace), best_pos, used, it


def _worker(rank, world, port, result_dir, case):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, D, lo, hi, seed, kind = case[:6]
    run = _replica_run if len(case) > 6 and case[6] == "replica" else _sharded_run
    tr, bp, used, it = run(rank, world, cfg, np.full(D, lo), np.full(D, hi), seed, kind)
    np.savez(os.path.join(result_dir, f"r{rank}.npz"), trace=tr, best_pos=bp, used=used, it=it)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("kind", [O.OBJ_SPHERE, O.OBJ_RASTRIGIN])
def test_two_rank_sharded_run_matches_unsharded(tmp_path, kind):
    import torch.multiprocessing as mp

    cfg = O.Config(batches=1, fireworks=4, sparks_per_firework=12, guides_per_firework=2, guide_fraction=0.25,
                   boosts=[1.0, 2.0], max_evaluations=4 + 25 * 4 * 14)
    D, lo, hi, seed = 6, -5.12, 5.12, 17
    case = (cfg, D, lo, hi, seed, kind)
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), case), nprocs=2, join=True)
    ref = O.Oracle().run(cfg, np.full(D, lo), np.full(D, hi), O.ObjectiveDesc(kind=kind), seed)
    for r in range(2):
        got = np.load(tmp_path / f"r{r}.npz")
        assert got["trace"].shape[0] == ref.trace_best.shape[1]
        assert np.array_equal(got["trace"][:, 1], ref.trace_best[0])
        assert np.array_equal(got["trace"][:, 0].astype(np.uint64), ref.trace_evals[0])
        assert np.array_equal(got["best_pos"], ref.best_position)
        assert int(got["used"]) == ref.evaluations_used and int(got["it"]) == ref.iterations


@pytest.mark.parametrize("kind", [O.OBJ_SPHERE, O.OBJ_RASTRIGIN])
def test_two_rank_replica_run_matches_unsharded(tmp_path, kind):
    import torch.multiprocessing as mp

    cfg = O.Config(batches=2, fireworks=4, sparks_per_firework=12, guides_per_firework=2, guide_fraction=0.25,
                   boosts=[1.0, 2.0], max_evaluations=8 + 25 * 2 * 4 * 14)
    D, lo, hi, seed = 6, -5.12, 5.12, 23
    case = (cfg, D, lo, hi, seed, kind, "replica")
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), case), nprocs=2, join=True)
    ref = O.Oracle().run(cfg, np.full(D, lo), np.full(D, hi), O.ObjectiveDesc(kind=kind), seed)
    assert ref.losers_reinitialized > 0
    for r in range(2):
        got = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(got["trace"][:, 1], ref.trace_best[r])
        assert np.array_equal(got["trace"][:, 0].astype(np.uint64), ref.trace_evals[r])
        assert np.array_equal(got["best_pos"], ref.best_position[r])
        assert int(got["used"]) == ref.evaluations_used and int(got["it"]) == ref.iterations
