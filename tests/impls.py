"""Two implementations behind one test interface, so the reference's own
known-answer tests (tests/test_*.cpp of the reference) run against both the
CPU oracle (fp64 restatement) and the B200 engine (fp32 state)."""
from __future__ import annotations

import numpy as np

import oracle as O


class OracleImpl:
    name = "oracle"
    exact = True  # fp64, bit-identical to the reference

    def __init__(self):
        self.o = O.Oracle()

    def initialize(self, cfg: O.Config, lower, upper, seed, kind=O.OBJ_SPHERE):
        pos = self.o.initialize_positions(cfg, lower, upper, seed)
        fit, _ = self.o.batched_apply(O.ObjectiveDesc(kind=kind), pos)
        amp_ = cfg.initial_amplitude if cfg.initial_amplitude > 0 else 0.5 * float(np.max(np.asarray(upper) - np.asarray(lower)))
        return pos, fit, np.full(fit.shape, amp_)

    def explode(self, pos, amp, lam, it, seed):
        return self.o.explode(pos, amp, lam, it, seed)

    def random_mapping(self, cand, per, pos, lower, upper, it, seed, stream):
        return self.o.random_mapping(cand, per, pos, lower, upper, it, seed, stream)

    def guiding_vector(self, sparks, fit, lam, top):
        return self.o.guiding_vector(sparks, fit, lam, top)

    def multi_guiding_sparks(self, pos, delta, boosts):
        return self.o.multi_guiding_sparks(pos, delta, boosts)

    def select_best(self, pos, fit, sparks, sfit, lam, guides=None, gfit=None, M=0):
        return self.o.select_best(pos, fit, sparks, sfit, lam, guides, gfit, M)

    def update_amplitudes(self, amp, improved, Ca, Cr, max_range):
        return self.o.update_amplitudes(amp, improved, Ca, Cr, max_range)

    def loser_out(self, pos, fit, amp, li, used, cfg, lower, upper, it, seed, iters_rem, kind=O.OBJ_SPHERE):
        p, f, a, l, n = self.o.loser_out(pos, fit, amp, li, cfg, lower, upper, it, seed, iters_rem,
                                         O.ObjectiveDesc(kind=kind))
        return p, f, a, l, n, used + n

    def run(self, cfg, lower, upper, kind, seed):
        return self.o.run(cfg, lower, upper, O.ObjectiveDesc(kind=kind), seed)

    def batched_apply(self, kind, rows):
        return self.o.batched_apply(O.ObjectiveDesc(kind=kind), rows)

    def argmin(self, fitness):
        return self.o.argmin_per_population(fitness)


class GpuImpl:
    name = "gpu"
    exact = False  # fp32 positions: results are the fp32 image of the reference's

    def __init__(self):
        import paper_2501_03944_b200 as P

        self.P = P

    def _cfg(self, cfg: O.Config):
        return self.P.MgfwaConfig(**cfg.__dict__)

    def _obj(self, kind):
        P = self.P
        return {O.OBJ_SPHERE: P.Sphere(), O.OBJ_RASTRIGIN: P.Rastrigin(), O.OBJ_ACKLEY: P.Ackley()}[kind]

    def initialize(self, cfg, lower, upper, seed, kind=O.OBJ_SPHERE):
        st = self.P.initialize(self._cfg(cfg), self.P.SearchSpace(lower, upper), seed, self._obj(kind))
        return st.positions, st.fitness, st.amplitudes

    def explode(self, pos, amp, lam, it, seed):
        pos = np.asarray(pos, dtype=np.float64)
        B, mu, D = pos.shape
        st = self.P.FireworkState(pos, np.zeros((B, mu)), np.asarray(amp, dtype=np.float64), np.zeros((B, mu)))
        cfg = self.P.MgfwaConfig(batches=B, fireworks=mu, sparks_per_firework=lam, max_evaluations=1)
        return self.P.explode(st, cfg, it, seed).positions

    def random_mapping(self, cand, per, pos, lower, upper, it, seed, stream):
        pos = np.asarray(pos, dtype=np.float64)
        B, mu, D = pos.shape
        st = self.P.FireworkState(pos, np.zeros((B, mu)), np.ones((B, mu)), np.zeros((B, mu)))
        cs = self.P.CandidateSet(per, np.asarray(cand, dtype=np.float64))
        return self.P.random_mapping(cs, st, self.P.SearchSpace(lower, upper), it, seed, stream).positions

    def guiding_vector(self, sparks, fit, lam, top):
        sparks = np.asarray(sparks, dtype=np.float64)
        B, rows, D = sparks.shape
        sigma = (top - 0.5) / lam  # ceil(sigma * lam) == top exactly
        cfg = self.P.MgfwaConfig(batches=B, fireworks=rows // lam, sparks_per_firework=lam,
                                 guide_fraction=sigma, max_evaluations=1)
        return self.P.guiding_vector(self.P.CandidateSet(lam, sparks, np.asarray(fit, dtype=np.float64)), cfg)

    def multi_guiding_sparks(self, pos, delta, boosts):
        pos = np.asarray(pos, dtype=np.float64)
        B, mu, D = pos.shape
        st = self.P.FireworkState(pos, np.zeros((B, mu)), np.ones((B, mu)), np.zeros((B, mu)))
        cfg = self.P.MgfwaConfig(batches=B, fireworks=mu, guides_per_firework=len(boosts), boosts=list(boosts),
                                 max_evaluations=1)
        return self.P.multi_guiding_sparks(st, delta, cfg).positions

    def select_best(self, pos, fit, sparks, sfit, lam, guides=None, gfit=None, M=0):
        pos = np.asarray(pos, dtype=np.float64)
        B, mu, D = pos.shape
        st = self.P.FireworkState(pos, np.asarray(fit, dtype=np.float64), np.ones((B, mu)), np.zeros((B, mu)))
        sp = self.P.CandidateSet(lam, np.asarray(sparks, dtype=np.float64), np.asarray(sfit, dtype=np.float64))
        gs = None
        if guides is not None and M > 0:
            gs = self.P.CandidateSet(M, np.asarray(guides, dtype=np.float64), np.asarray(gfit, dtype=np.float64))
        r = self.P.select_best(st, sp, gs)
        return r.state.positions, r.state.fitness, r.state.last_improvement, r.improved

    def update_amplitudes(self, amp, improved, Ca, Cr, max_range):
        cfg = self.P.MgfwaConfig(amp_amplify=Ca, amp_reduce=Cr, max_evaluations=1)
        return self.P.update_amplitudes(amp, improved, cfg, max_range)

    def loser_out(self, pos, fit, amp, li, used, cfg, lower, upper, it, seed, iters_rem, kind=O.OBJ_SPHERE):
        st = self.P.FireworkState(np.asarray(pos, dtype=np.float64), np.asarray(fit, dtype=np.float64),
                                  np.asarray(amp, dtype=np.float64), np.asarray(li, dtype=np.float64), used)
        n = self.P.loser_out(st, self._cfg(cfg), self.P.SearchSpace(lower, upper), it, seed, iters_rem,
                             self._obj(kind))
        return st.positions, st.fitness, st.amplitudes, st.last_improvement, n, st.evaluations_used

    def run(self, cfg, lower, upper, kind, seed):
        r = self.P.run(self._cfg(cfg), self.P.SearchSpace(lower, upper), self._obj(kind), seed)
        r.trace_evals = r.trace_evaluations
        return r

    def batched_apply(self, kind, rows):
        return self.P.batched_apply(self._obj(kind), rows)

    def argmin(self, fitness):
        return self.P.argmin_per_population(fitness)


def f32(a):
    """fp32 image of an fp64 array (what a float32 engine stores)."""
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)
