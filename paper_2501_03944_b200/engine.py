"""Python mirror of the reference's optimizer / objective interface over the
B200 engine's C-ABI (include/mgfwa_b200.h).

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/mgfwa/{config,engine,backend}.hpp):
``MgfwaConfig``, ``SearchSpace``, ``FireworkState``, ``CandidateSet``,
``RunRecord``, ``run()`` and the operators ``initialize``, ``explode``,
``random_mapping``, ``guiding_vector``, ``multi_guiding_sparks``,
``select_best``, ``update_amplitudes``, ``loser_out``, ``batched_apply``,
``argmin_per_population``.  ``std::invalid_argument`` surfaces as
``ValueError`` with the reference's message.  Every call runs on the GPU;
there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi as A

# RngStream, rng.hpp:11-18
kInit, kExplode, kMapping, kGuide, kReinit, kWeights = 1, 2, 3, 4, 5, 6


class CudaError(RuntimeError):
    pass


def _check(rc: int, ctx=None):
    if rc == A.MGFWA_OK:
        return
    msg = A.lib().mgfwa_last_error(ctx)
    msg = msg.decode() if msg else f"mgfwa error {rc}"
    if rc == A.MGFWA_EINVAL:
        raise ValueError(msg)
    raise CudaError(msg)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _pd(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _pu64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


# ------------------------------------------------------------------ config
@dataclass
class MgfwaConfig:
    """MgfwaConfig, config.hpp:33-67 (same fields, same defaults)."""

    batches: int = 8
    fireworks: int = 5
    sparks_per_firework: int = 30
    guides_per_firework: int = 3
    guide_fraction: float = 0.2
    boosts: Sequence[float] = field(default_factory=lambda: [1.0, 2.0, 4.0])
    amp_amplify: float = 1.2
    amp_reduce: float = 0.9
    initial_amplitude: float = 0.0
    max_evaluations: int = 0
    wall_clock_budget_ms: float = 0.0

    def validate(self) -> None:
        """MgfwaConfig::validate (config.cpp:42-79): raises ValueError with the
        reference's message."""
        c, _keep = self._c()
        _check(A.lib().mgfwa_validate_config(C.byref(c)))

    def top_spark_count(self) -> int:  # config.cpp:37-40
        return int(math.ceil(self.guide_fraction * float(self.sparks_per_firework)))

    def evaluations_per_wave(self) -> int:  # config.hpp:55-58
        return self.batches * self.fireworks * (self.sparks_per_firework + self.guides_per_firework)

    def resolved_initial_amplitude(self, max_range: float) -> float:  # config.hpp:61-63
        return self.initial_amplitude if self.initial_amplitude > 0.0 else 0.5 * max_range

    def _c(self):
        boosts = _f64(list(self.boosts) if len(self.boosts) else [0.0])
        c = A.mgfwa_config_t(self.batches, self.fireworks, self.sparks_per_firework,
                             self.guides_per_firework, self.guide_fraction, _pd(boosts),
                             len(self.boosts), self.amp_amplify, self.amp_reduce,
                             self.initial_amplitude, self.max_evaluations, self.wall_clock_budget_ms)
        return c, boosts


@dataclass
class SearchSpace:
    """SearchSpace, config.hpp:11-28."""

    lower: np.ndarray
    upper: np.ndarray

    def __post_init__(self):
        self.lower = _f64(self.lower).reshape(-1)
        self.upper = _f64(self.upper).reshape(-1)

    @staticmethod
    def box(dim: int, lo: float, hi: float) -> "SearchSpace":
        return SearchSpace(np.full(dim, lo), np.full(dim, hi))

    def dim(self) -> int:
        return int(self.lower.size)

    def max_range(self) -> float:
        return float(np.max(self.upper - self.lower)) if self.dim() else 0.0

    def contains(self, d: int, x: float) -> bool:
        return bool(x >= self.lower[d] and x <= self.upper[d])

    def _c(self):
        return A.mgfwa_space_t(_pd(self.lower), _pd(self.upper), self.lower.size)


# --------------------------------------------------------------- objectives
@dataclass(frozen=True)
class Objective:
    """Closed objective descriptor replacing the host std::function
    Objective of backend.hpp:15 (evaluated on the device)."""

    kind: int
    in_dim: int = 0
    hidden: int = 0
    out_dim: int = 0
    samples: int = 0
    data_seed: int = 0
    net_id: int = 0
    weight_seed: int = 0

    def dim(self, analytic_dim: int = 0) -> int:
        if self.kind == A.OBJ_MLP_WEIGHTS:
            return self.hidden * self.in_dim + self.hidden + self.out_dim * self.hidden + self.out_dim
        if self.kind == A.OBJ_LENET:
            return LENET_DIM
        if self.kind == A.OBJ_NET:
            return NET_REGISTRY[self.net_id][2]
        return analytic_dim

    def _c(self):
        return A.mgfwa_objective_t(self.kind, self.in_dim, self.hidden, self.out_dim, self.samples,
                                   self.data_seed, self.net_id, self.weight_seed)


def Sphere() -> Objective:  # nets.cpp:80-84
    return Objective(A.OBJ_SPHERE)


def Rastrigin() -> Objective:
    return Objective(A.OBJ_RASTRIGIN)


def Ackley() -> Objective:
    return Objective(A.OBJ_ACKLEY)


def MlpWeights(in_dim: int = 784, hidden: int = 32, out_dim: int = 10, samples: int = 1024,
               data_seed: int = 1) -> Objective:
    """Mean CE of an I-H-O ReLU MLP whose weights (W1,b1,W2,b2 in reference
    Layer order) are the candidate; bf16 tensor-core evaluation."""
    return Objective(A.OBJ_MLP_WEIGHTS, in_dim, hidden, out_dim, samples, data_seed)


# net_registry(), nets.cpp:36-55: id -> (scale, activation, input_dim,
# hidden_dim, hidden_layers, reported_params)
NET_REGISTRY = {
    1: ("small", "relu", 10, 16, 2, 465), 2: ("small", "gelu", 10, 32, 5, 4609),
    3: ("small", "relu", 20, 16, 5, 1441), 4: ("small", "gelu", 20, 32, 5, 4929),
    5: ("medium", "relu", 100, 64, 8, 35649), 6: ("medium", "gelu", 100, 128, 8, 128641),
    7: ("medium", "relu", 200, 64, 8, 42049), 8: ("medium", "gelu", 200, 128, 8, 141441),
    9: ("large", "relu", 1000, 256, 11, 914433), 10: ("large", "gelu", 1000, 512, 11, 3137585),
    11: ("large", "relu", 2000, 256, 11, 1173433), 12: ("large", "gelu", 2000, 512, 11, 3657585),
}


def Net(net_id: int, weight_seed: int = 1) -> Objective:
    """The reference's benchmark network net_id (MlpBlackBox(net_spec(id),
    weight_seed), nets.cpp:36-167): fixed weights, the candidate is the
    network input, scalar output; fp64 evaluation on the device."""
    if net_id not in NET_REGISTRY:
        raise ValueError("net id must be in 1..12")
    return Objective(A.OBJ_NET, net_id=net_id, weight_seed=weight_seed)


def net_param_count(net_id: int) -> int:
    """param_count(net_spec(id)), nets.cpp:64-72."""
    _, _, d, h, lh, _ = NET_REGISTRY[net_id]
    return (d * h + h) + (lh - 1) * (h * h + h) + (h + 1)


LENET_DIM = (6 * 25 + 6) + (16 * 6 * 25 + 16) + (400 * 120 + 120) + (120 * 84 + 84) + (84 * 10 + 10)


def LeNet(samples: int = 1024, data_seed: int = 1) -> Objective:
    """Mean CE of LeNet-5 (conv5x5 1->6 pad 2, ReLU, avgpool2, conv5x5 6->16,
    ReLU, avgpool2, fc 400-120-84-10) on S synthetic 28x28 samples; the
    61,706 parameters (PyTorch order, oracle f_lenet) are the candidate;
    bf16 tensor-core evaluation (config C3)."""
    return Objective(A.OBJ_LENET, 784, 0, 10, samples, data_seed)


# ------------------------------------------------------------------- state
@dataclass
class FireworkState:
    """FireworkState, engine.hpp:16-22 (positions [B][mu][D])."""

    positions: np.ndarray
    fitness: np.ndarray
    amplitudes: np.ndarray
    last_improvement: np.ndarray
    evaluations_used: int = 0


@dataclass
class CandidateSet:
    """CandidateSet, engine.hpp:27-43 (positions [B][mu*K][D])."""

    per_firework: int
    positions: np.ndarray
    fitness: Optional[np.ndarray] = None

    def fireworks(self) -> int:
        return self.positions.shape[1] // self.per_firework


@dataclass
class RunRecord:
    """RunRecord, engine.hpp:56-67; trace as [batch][wave] arrays."""

    config: MgfwaConfig
    space: SearchSpace
    seed: int
    trace_evaluations: np.ndarray
    trace_best: np.ndarray
    trace_wall_ms: np.ndarray
    best_position: np.ndarray
    best_fitness: np.ndarray
    evaluations_used: int
    iterations: int
    losers_reinitialized: int
    nan_evaluations: int


# ------------------------------------------------------------------ engine
class Engine:
    """One device-resident run: initialize(), step()/enqueue(), results."""

    SHARD_MODES = {"firework": 0, "replica": 1}  # MGFWA_SHARD_* (include/mgfwa_b200.h)

    def __init__(self, config: MgfwaConfig, space: SearchSpace, objective: Objective, seed: int,
                 device: int = 0, rank: int = 0, world: int = 1, shard_mode: str = "firework"):
        """shard_mode (world > 1): "firework" — fireworks split evenly, one
        all-gather of the selected state per generation; "replica" — each rank
        owns whole batches (needs batches % world == 0), the per-generation
        exchange is the loser count only, results are valid for the rank's own
        batches (`owned_batches`)."""
        self.config, self.space, self.objective, self.seed = config, space, objective, seed
        self.rank, self.world, self.shard_mode = rank, world, shard_mode
        if shard_mode not in self.SHARD_MODES:
            raise ValueError(f"shard_mode must be one of {sorted(self.SHARD_MODES)}")
        c, self._keep = config._c()
        sp = space._c()
        ob = objective._c()
        h = C.c_void_p()
        if world == 1:
            _check(A.lib().mgfwa_create(C.byref(c), C.byref(sp), C.byref(ob), seed, device, C.byref(h)))
        else:
            _check(A.lib().mgfwa_create_shard(C.byref(c), C.byref(sp), C.byref(ob), seed, device, rank, world,
                                              C.byref(h)))
        self.h = h
        if shard_mode != "firework":
            _check(A.lib().mgfwa_set_shard_mode(self.h, self.SHARD_MODES[shard_mode]), self.h)

    @property
    def owned_batches(self) -> range:
        """Batches whose trace / best / state this context holds (all of them
        except under replica sharding)."""
        B = self.config.batches
        if self.shard_mode != "replica":
            return range(B)
        return range(self.rank * B // self.world, (self.rank + 1) * B // self.world)

    # ---- firework sharding (one rank per GPU, NCCL all-gather per generation)
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(A.lib().mgfwa_nccl_unique_id(buf))
        return buf.raw

    def attach_nccl(self, unique_id: bytes):
        buf = C.create_string_buffer(unique_id, 128)
        _check(A.lib().mgfwa_attach_nccl(self.h, buf, self.world, self.rank), self.h)

    def phase(self, p: int):
        """Manual stepping (no NCCL): phase 1 = up to selection, 2 = loser-out .. record."""
        _check(A.lib().mgfwa_generation_phase(self.h, p), self.h)

    def import_shard(self, other: "Engine"):
        """In-process exchange: copy `other`'s owned fireworks into this replica."""
        _check(A.lib().mgfwa_shard_exchange(self.h, other.h), self.h)

    def close(self):
        if getattr(self, "h", None):
            A.lib().mgfwa_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int):
        _check(A.lib().mgfwa_set_stream(self.h, C.c_void_p(stream_handle)), self.h)

    def kernels_per_generation(self) -> int:
        n = C.c_uint64()
        _check(A.lib().mgfwa_kernels_per_generation(self.h, C.byref(n)), self.h)
        return int(n.value)

    def initialize(self):
        _check(A.lib().mgfwa_initialize(self.h), self.h)

    def time_fitness(self, iters: int = 10):
        """(ms per launch, candidates per launch) of the dominant kernel."""
        ms, units = C.c_double(), C.c_uint64()
        _check(A.lib().mgfwa_time_fitness(self.h, iters, C.byref(ms), C.byref(units)), self.h)
        return ms.value, int(units.value)

    KERNELS = {"fitness": 0, "explode": 1, "rank": 2, "guides": 3, "guide_fitness": 4, "select": 5}

    def time_kernel(self, kernel: str, iters: int = 10):
        """(ms per launch, rows per launch) of one generation kernel on the
        current state (mgfwa_time_kernel)."""
        ms, units = C.c_double(), C.c_uint64()
        _check(A.lib().mgfwa_time_kernel(self.h, self.KERNELS[kernel], iters, C.byref(ms), C.byref(units)),
               self.h)
        return ms.value, int(units.value)

    def step(self, max_generations: int) -> int:
        n = C.c_uint64()
        _check(A.lib().mgfwa_step(self.h, max_generations, C.byref(n)), self.h)
        return int(n.value)

    def enqueue(self, n: int):
        _check(A.lib().mgfwa_enqueue_generations(self.h, n), self.h)

    def sync(self):
        _check(A.lib().mgfwa_sync(self.h), self.h)

    def run(self) -> "RunRecord":
        cnt = A.mgfwa_counters_t()
        _check(A.lib().mgfwa_run(self.h, C.byref(cnt)), self.h)
        return self.record()

    def counters(self) -> dict:
        cnt = A.mgfwa_counters_t()
        _check(A.lib().mgfwa_get_counters(self.h, C.byref(cnt)), self.h)
        return {k: int(getattr(cnt, k)) for k, _ in A.mgfwa_counters_t._fields_}

    def best(self):
        B, D = self.config.batches, self.space.dim()
        bf, bp = np.empty(B), np.empty((B, D))
        _check(A.lib().mgfwa_get_best(self.h, _pd(bf), _pd(bp)), self.h)
        return bf, bp

    def state(self) -> FireworkState:
        B, mu, D = self.config.batches, self.config.fireworks, self.space.dim()
        pos, fit, amp, li = np.empty((B, mu, D)), np.empty((B, mu)), np.empty((B, mu)), np.empty((B, mu))
        _check(A.lib().mgfwa_get_state(self.h, _pd(pos), _pd(fit), _pd(amp), _pd(li)), self.h)
        return FireworkState(pos, fit, amp, li, self.counters()["evaluations_used"])

    def candidates(self, bf16: bool = False):
        """The last generation's mapped sparks / guides and their fitness
        (mgfwa_get_candidates): (sparks [Fl*lam][D], spark_fitness,
        guides [Fl*M][D] or None, guide_fitness or None, bf16 shadow as
        uint16 [Fl*lam][D] or None)."""
        cfg = self.config
        Fl = cfg.batches * cfg.fireworks // self.world
        D = self.space.dim()
        sp, sf = np.empty((Fl * cfg.sparks_per_firework, D)), np.empty(Fl * cfg.sparks_per_firework)
        M = cfg.guides_per_firework
        gd, gf = (np.empty((Fl * M, D)), np.empty(Fl * M)) if M else (None, None)
        sh = np.empty((Fl * cfg.sparks_per_firework, D), dtype=np.uint16) if bf16 else None
        _check(A.lib().mgfwa_get_candidates(
            self.h, _pd(sp), _pd(sf), _pd(gd) if M else None, _pd(gf) if M else None,
            sh.ctypes.data_as(C.POINTER(C.c_uint16)) if bf16 else None), self.h)
        return sp, sf, gd, gf, sh

    def record(self) -> RunRecord:
        cnt = self.counters()
        B = self.config.batches
        waves = C.c_uint64()
        _check(A.lib().mgfwa_get_trace(self.h, None, None, None, 0, C.byref(waves)), self.h)
        w = int(waves.value)
        te, tb, tw = np.zeros((B, w), dtype=np.uint64), np.zeros((B, w)), np.zeros((B, w))
        if w:
            _check(A.lib().mgfwa_get_trace(self.h, _pu64(te), _pd(tb), _pd(tw), w, None), self.h)
        bf, bp = self.best()
        return RunRecord(self.config, self.space, self.seed, te, tb, tw, bp, bf, cnt["evaluations_used"],
                         cnt["iterations"], cnt["losers_reinitialized"], cnt["nan_evaluations"])


def run(config: MgfwaConfig, space: SearchSpace, objective: Objective, seed: int,
        device: int = 0) -> RunRecord:
    """run(), engine.cpp:313-423, on the B200 engine."""
    eng = Engine(config, space, objective, seed, device)
    try:
        return eng.run()
    finally:
        eng.close()


# ---------------------------------------------------------------- operators
def _wide(dim: int) -> SearchSpace:
    return SearchSpace(np.full(dim, -3.0e38), np.full(dim, 3.0e38))


def initialize(config: MgfwaConfig, space: SearchSpace, seed: int, objective: Objective) -> FireworkState:
    """initialize(), engine.cpp:45-76."""
    B, mu, D = config.batches, config.fireworks, space.dim()
    pos, fit, amp = np.empty((B, mu, D)), np.empty((B, mu)), np.empty((B, mu))
    c, keep = config._c()
    sp, ob = space._c(), objective._c()
    _check(A.lib().mgfwa_op_initialize(C.byref(c), C.byref(sp), C.byref(ob), seed, _pd(pos), _pd(fit),
                                       _pd(amp)))
    return FireworkState(pos, fit, amp, np.zeros((B, mu)), B * mu)


def explode_map(state: FireworkState, config: MgfwaConfig, space: SearchSpace, iteration: int,
                seed: int) -> CandidateSet:
    """random_mapping(explode(state), kMapping) (engine.cpp:78-131), fused."""
    pos, amp = _f64(state.positions), _f64(state.amplitudes)
    B, mu, D = pos.shape
    cfg = MgfwaConfig(**{**config.__dict__, "batches": B, "fireworks": mu})
    c, keep = cfg._c()
    sp = space._c()
    out = np.empty((B, mu * cfg.sparks_per_firework, D))
    _check(A.lib().mgfwa_op_explode_map(C.byref(c), C.byref(sp), _pd(pos), _pd(amp), iteration, seed,
                                        _pd(out)))
    return CandidateSet(cfg.sparks_per_firework, out, None)


def explode(state: FireworkState, config: MgfwaConfig, iteration: int, seed: int) -> CandidateSet:
    """explode(), engine.cpp:78-101 (no repair: unbounded box)."""
    return explode_map(state, config, _wide(state.positions.shape[2]), iteration, seed)


def random_mapping(candidates: CandidateSet, state: FireworkState, space: SearchSpace, iteration: int,
                   seed: int, stream: int) -> CandidateSet:
    """random_mapping(), engine.cpp:103-131."""
    cand, pos = _f64(candidates.positions), _f64(state.positions)
    B, rows, D = cand.shape
    out = np.empty_like(cand)
    sp = space._c()
    _check(A.lib().mgfwa_op_random_mapping(C.byref(sp), _pd(cand), B, rows, candidates.per_firework,
                                           _pd(pos), pos.shape[1], iteration, seed, stream, _pd(out)))
    return CandidateSet(candidates.per_firework, out, candidates.fitness)


def guiding_vector(sparks: CandidateSet, config: MgfwaConfig) -> np.ndarray:
    """guiding_vector(), engine.cpp:133-172 -> delta [B][mu][D] (fp32-rounded)."""
    if config.sparks_per_firework < 2 * config.top_spark_count():
        raise ValueError("guiding_vector: elite and poor sets overlap")
    if sparks.fitness is None:
        raise ValueError("guiding_vector: sparks not evaluated")
    s, f = _f64(sparks.positions), _f64(sparks.fitness)
    B, rows, D = s.shape
    mu = rows // sparks.per_firework
    cfg = MgfwaConfig(**{**config.__dict__, "batches": B, "fireworks": mu,
                         "sparks_per_firework": sparks.per_firework})
    c, keep = cfg._c()
    out = np.empty((B, mu, D))
    _check(A.lib().mgfwa_op_guiding_vector(C.byref(c), D, _pd(s), _pd(f), _pd(out)))
    return out


def guides_map(state: FireworkState, sparks: CandidateSet, config: MgfwaConfig, space: SearchSpace,
               iteration: int, seed: int) -> CandidateSet:
    """random_mapping(multi_guiding_sparks(state, guiding_vector(sparks)),
    kGuide) (engine.cpp:379-382), fused as in the generation loop."""
    pos, s, f = _f64(state.positions), _f64(sparks.positions), _f64(sparks.fitness)
    B, mu, D = pos.shape
    cfg = MgfwaConfig(**{**config.__dict__, "batches": B, "fireworks": mu})
    c, keep = cfg._c()
    sp = space._c()
    out = np.empty((B, mu * cfg.guides_per_firework, D))
    _check(A.lib().mgfwa_op_guides(C.byref(c), C.byref(sp), _pd(pos), _pd(s), _pd(f), iteration, seed,
                                   _pd(out)))
    return CandidateSet(cfg.guides_per_firework, out, None)


def multi_guiding_sparks(state: FireworkState, delta: np.ndarray, config: MgfwaConfig) -> CandidateSet:
    """multi_guiding_sparks(), engine.cpp:174-196, through the production
    guide kernel: sparks {delta, 0} with lambda = 2, top = 1 give exactly
    delta as the guiding vector; the box is unbounded (no repair)."""
    pos, dl = _f64(state.positions), _f64(delta)
    B, mu, D = pos.shape
    sparks = np.zeros((B, mu * 2, D))
    sparks[:, 0::2, :] = dl
    fit = np.tile(np.array([0.0, 1.0]), (B, mu))
    cfg = MgfwaConfig(**{**config.__dict__, "batches": B, "fireworks": mu, "sparks_per_firework": 2,
                         "guide_fraction": 0.5})
    return guides_map(state, CandidateSet(2, sparks, fit), cfg, _wide(D), 1, 0)


@dataclass
class SelectionResult:
    state: FireworkState
    improved: np.ndarray
    amplitudes_after_update: np.ndarray


def select_best(state: FireworkState, sparks: CandidateSet, guides: Optional[CandidateSet],
                config: Optional[MgfwaConfig] = None, max_range: float = 1.0) -> SelectionResult:
    """select_best(), engine.cpp:198-242 (+ update_amplitudes with
    ``config``/``max_range``, engine.cpp:244-256, as the fused kernel does)."""
    pos, fit, amp = _f64(state.positions), _f64(state.fitness), _f64(state.amplitudes)
    B, mu, D = pos.shape
    base = config or MgfwaConfig()
    M = guides.per_firework if guides is not None else 0
    cfg = MgfwaConfig(**{**base.__dict__, "batches": B, "fireworks": mu,
                         "sparks_per_firework": sparks.per_firework, "guides_per_firework": M,
                         "boosts": [1.0] + [2.0] * (M - 1) if M else []})
    c, keep = cfg._c()
    space = SearchSpace(np.zeros(D), np.full(D, max_range))
    sp = space._c()
    s, sf = _f64(sparks.positions), _f64(sparks.fitness)
    if guides is not None:
        g, gf = _f64(guides.positions), _f64(guides.fitness)
        gp, gfp = _pd(g), _pd(gf)
    else:
        gp = gfp = None
    npos, nfit, nli, imp, namp = (np.empty_like(pos), np.empty((B, mu)), np.empty((B, mu)),
                                  np.empty((B, mu)), np.empty((B, mu)))
    _check(A.lib().mgfwa_op_select_best(C.byref(c), C.byref(sp), _pd(pos), _pd(fit), _pd(amp), _pd(s),
                                        _pd(sf), gp, gfp, _pd(npos), _pd(nfit), _pd(nli), _pd(imp),
                                        _pd(namp)))
    return SelectionResult(FireworkState(npos, nfit, amp.copy(), nli, state.evaluations_used), imp, namp)


def update_amplitudes(amplitudes: np.ndarray, improved: np.ndarray, config: MgfwaConfig,
                      max_range: float) -> np.ndarray:
    """update_amplitudes(), engine.cpp:244-256, via the fused select kernel:
    one spark per firework that improves (fitness 0 < 1) or not (2 > 1)."""
    a, im = _f64(amplitudes), _f64(improved)
    shape = a.shape
    a2, im2 = a.reshape(1, -1), im.reshape(1, -1)
    n = a2.shape[1]
    st = FireworkState(np.zeros((1, n, 1)), np.ones((1, n)), a2, np.zeros((1, n)))
    sp = CandidateSet(1, np.zeros((1, n, 1)), np.where(im2 != 0.0, 0.0, 2.0))
    res = select_best(st, sp, None, config, max_range)
    return res.amplitudes_after_update.reshape(shape)


def loser_out(state: FireworkState, config: MgfwaConfig, space: SearchSpace, iteration: int, seed: int,
              iterations_remaining: float, objective: Objective) -> int:
    """loser_out(), engine.cpp:258-311; updates ``state`` in place and
    returns the number of reinitialized fireworks."""
    pos = _f64(state.positions).copy()
    fit, amp, li = (_f64(x).copy() for x in (state.fitness, state.amplitudes, state.last_improvement))
    B, mu, D = pos.shape
    cfg = MgfwaConfig(**{**config.__dict__, "batches": B, "fireworks": mu})
    c, keep = cfg._c()
    sp, ob = space._c(), objective._c()
    used = C.c_uint64(state.evaluations_used)
    n = C.c_uint64()
    _check(A.lib().mgfwa_op_loser_out(C.byref(c), C.byref(sp), C.byref(ob), _pd(pos), _pd(fit), _pd(amp),
                                      _pd(li), C.byref(used), iteration, seed, iterations_remaining,
                                      C.byref(n)))
    state.positions, state.fitness, state.amplitudes, state.last_improvement = pos, fit, amp, li
    state.evaluations_used = int(used.value)
    return int(n.value)


def batched_apply(objective: Objective, candidates) -> tuple:
    """batched_apply(), backend.cpp:28-67: returns (fitness [.. x N], nan_flagged)."""
    x = _f64(candidates)
    D = x.shape[-1]
    flat = np.ascontiguousarray(x.reshape(-1, D))
    out = np.empty(flat.shape[0])
    nan = C.c_uint64()
    _check(A.lib().mgfwa_op_batched_apply(C.byref(objective._c()), _pd(flat), flat.shape[0], D, _pd(out),
                                          C.byref(nan)))
    return out.reshape(x.shape[:-1]), int(nan.value)


def argmin_per_population(fitness: np.ndarray):
    """argmin_per_population(), backend.cpp:69-83 -> (index, value)."""
    f = _f64(fitness)
    idx, val = np.empty(f.shape[0], dtype=np.uint64), np.empty(f.shape[0])
    _check(A.lib().mgfwa_op_argmin_per_population(_pd(f), f.shape[0], f.shape[1], _pu64(idx), _pd(val)))
    return idx, val


def key_hash(keys: np.ndarray) -> np.ndarray:
    """key_hash(), rng.hpp:43-52, evaluated on the device for keys [n][7]."""
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1, 7))
    out = np.empty(k.shape[0], dtype=np.uint64)
    _check(A.lib().mgfwa_key_hash(_pu64(k), k.shape[0], _pu64(out)))
    return out
