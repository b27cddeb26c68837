"""TEST INFRASTRUCTURE ONLY — ctypes front-ends for the two CPU checkers.

* ``Oracle`` wraps ``oracle/build/libmgfwa_oracle.so``: the plain-C fp64
  restatement of the reference generation path (oracle/mgfwa_oracle.c).
* ``Reference`` wraps ``oracle/_ref/libmgfwa_ref.so``: the UNMODIFIED
  reference engine (/root/reference/proj/src/{backend,config,engine,nets}.cpp)
  compiled by oracle/Makefile, behind the extern "C" seam oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
``--impl reference`` arm) may import this package, and only as the checker /
the CPU baseline.  The product package (paper_2501_03944_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libmgfwa_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmgfwa_ref.so")
REF_SRC = "/root/reference/proj"

# RngStream (rng.hpp:11-18) + kData
K_INIT, K_EXPLODE, K_MAPPING, K_GUIDE, K_REINIT, K_WEIGHTS, K_DATA = 1, 2, 3, 4, 5, 6, 7
OBJ_SPHERE, OBJ_RASTRIGIN, OBJ_ACKLEY, OBJ_MLP_WEIGHTS, OBJ_LENET, OBJ_NET = 1, 2, 3, 4, 5, 6

_u64 = C.c_uint64
_dbl = C.c_double
_pd = C.POINTER(C.c_double)
_pu64 = C.POINTER(C.c_uint64)


def build(with_reference: Optional[bool] = None) -> None:
    """Compile the C restatement (always) and oracle/_ref (when the reference
    sources are present, i.e. in the build container)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if with_reference is None:
        with_reference = os.path.isdir(REF_SRC)
    if with_reference:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _arr(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_pd)


@dataclass
class Config:
    """MgfwaConfig, config.hpp:33-47 (defaults identical)."""

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

    def top_spark_count(self) -> int:
        import math

        return int(math.ceil(self.guide_fraction * float(self.sparks_per_firework)))

    def evaluations_per_wave(self) -> int:
        return self.batches * self.fireworks * (self.sparks_per_firework + self.guides_per_firework)


class _CConfig(C.Structure):
    _fields_ = [
        ("batches", _u64), ("fireworks", _u64), ("sparks", _u64), ("guides", _u64),
        ("guide_fraction", _dbl), ("boosts", _pd), ("n_boosts", _u64),
        ("amp_amplify", _dbl), ("amp_reduce", _dbl), ("initial_amplitude", _dbl),
        ("max_evaluations", _u64), ("wall_clock_budget_ms", _dbl),
    ]


def _cconfig(cfg: Config):
    boosts = _arr(list(cfg.boosts) if len(cfg.boosts) else [0.0])
    c = _CConfig(cfg.batches, cfg.fireworks, cfg.sparks_per_firework, cfg.guides_per_firework,
                 cfg.guide_fraction, _p(boosts), len(cfg.boosts), cfg.amp_amplify,
                 cfg.amp_reduce, cfg.initial_amplitude, cfg.max_evaluations,
                 cfg.wall_clock_budget_ms)
    return c, boosts  # keep boosts alive


@dataclass
class ObjectiveDesc:
    kind: int = OBJ_SPHERE
    in_dim: int = 784
    hidden: int = 32
    out_dim: int = 10
    samples: int = 1024
    data_seed: int = 1
    net_id: int = 1
    weight_seed: int = 1

    def dim(self, analytic_dim: int = 0) -> int:
        if self.kind == OBJ_MLP_WEIGHTS:
            return self.hidden * self.in_dim + self.hidden + self.out_dim * self.hidden + self.out_dim
        if self.kind == OBJ_LENET:
            return 61706
        return analytic_dim


class _CObjDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("in_dim", C.c_uint32), ("hidden", C.c_uint32),
                ("out_dim", C.c_uint32), ("samples", C.c_uint32), ("data_seed", _u64),
                ("net_id", C.c_int), ("weight_seed", _u64)]


def _cobj(o: ObjectiveDesc) -> _CObjDesc:
    return _CObjDesc(o.kind, o.in_dim, o.hidden, o.out_dim, o.samples, o.data_seed,
                     o.net_id, o.weight_seed)


class _Counters(C.Structure):
    _fields_ = [("evaluations_used", _u64), ("iterations", _u64),
                ("losers_reinitialized", _u64), ("nan_evaluations", _u64), ("waves", _u64)]


@dataclass
class Record:
    """RunRecord, engine.hpp:56-67 (trace as [batch][wave] arrays)."""

    best_fitness: np.ndarray
    best_position: np.ndarray
    trace_evals: np.ndarray
    trace_best: np.ndarray
    trace_wall_ms: np.ndarray
    evaluations_used: int
    iterations: int
    losers_reinitialized: int
    nan_evaluations: int


def _trace_cap(cfg: Config) -> int:
    if cfg.max_evaluations == 0:
        return 1 << 16
    wave = max(cfg.evaluations_per_wave(), 1)
    return int(cfg.max_evaluations // wave + 3)


class Oracle:
    """ctypes wrapper of the C restatement (oracle/mgfwa_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(with_reference=False)
        L = self.lib = C.CDLL(path)
        L.orc_key_hash.restype = _u64
        L.orc_key_hash.argtypes = [_u64] * 7
        L.orc_unit_uniform.restype = _dbl
        L.orc_unit_uniform.argtypes = [_u64] * 7
        L.orc_config_validate.restype = C.c_char_p
        L.orc_config_validate.argtypes = [C.POINTER(_CConfig)]
        L.orc_space_validate.restype = C.c_char_p
        L.orc_space_validate.argtypes = [_pd, _pd, _u64]
        L.orc_top_spark_count.restype = _u64
        L.orc_objective_create.restype = C.c_void_p
        L.orc_objective_create.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _u64]
        L.orc_objective_destroy.argtypes = [C.c_void_p]
        L.orc_objective_eval.restype = _dbl
        L.orc_objective_eval.argtypes = [C.c_void_p, _pd, _u64]
        L.orc_objective_data.restype = _pd
        L.orc_objective_data.argtypes = [C.c_void_p]
        L.orc_objective_labels.restype = C.POINTER(C.c_int32)
        L.orc_objective_labels.argtypes = [C.c_void_p]
        L.orc_batched_apply.restype = _u64
        L.orc_batched_apply.argtypes = [C.c_void_p, _pd, _u64, _u64, _pd]
        L.orc_argmin_per_population.argtypes = [_pd, _u64, _u64, _pu64, _pd]
        L.orc_population_range.argtypes = [_pd, _u64, _u64, _u64, _pd, _pd]
        L.orc_initialize_positions.argtypes = [C.POINTER(_CConfig), _pd, _pd, _u64, _u64, _pd]
        L.orc_explode.argtypes = [_pd, _pd, _u64, _u64, _u64, _u64, _u64, _u64, _pd]
        L.orc_random_mapping.argtypes = [_pd, _u64, _u64, _u64, _u64, _pd, _u64, _pd, _pd, _u64, _u64, _u64]
        L.orc_guiding_vector.restype = C.c_int
        L.orc_guiding_vector.argtypes = [_pd, _pd, _u64, _u64, _u64, _u64, _u64, _pd]
        L.orc_multi_guiding_sparks.argtypes = [_pd, _pd, _u64, _u64, _u64, _pd, _u64, _pd]
        L.orc_select_best.argtypes = [_pd, _pd, _u64, _u64, _u64, _pd, _pd, _u64, _pd, _pd, _u64, _pd, _pd, _pd, _pd]
        L.orc_update_amplitudes.argtypes = [_pd, _pd, _u64, _dbl, _dbl, _dbl, _pd]
        L.orc_loser_out.restype = _u64
        L.orc_loser_out.argtypes = [_pd, _pd, _pd, _pd, _u64, _u64, _u64, C.POINTER(_CConfig), _pd, _pd,
                                    _u64, _u64, _dbl, C.c_void_p, _pu64]
        L.orc_run.restype = C.c_char_p
        L.orc_run.argtypes = [C.POINTER(_CConfig), _pd, _pd, _u64, C.c_void_p, _u64, _pd, _pd, _pu64,
                              _pd, _pd, _u64, C.POINTER(_Counters)]
        self._objs = {}

    # -- rng
    def key_hash(self, seed, stream, it, b, n, k, d) -> int:
        return int(self.lib.orc_key_hash(seed, stream, it, b, n, k, d))

    def unit_uniform(self, seed, stream, it, b, n, k, d) -> float:
        return float(self.lib.orc_unit_uniform(seed, stream, it, b, n, k, d))

    # -- config
    def validate(self, cfg: Config) -> Optional[str]:
        c, keep = _cconfig(cfg)
        r = self.lib.orc_config_validate(C.byref(c))
        return None if r is None else r.decode()

    # -- objectives
    def objective(self, desc: ObjectiveDesc):
        key = (desc.kind, desc.in_dim, desc.hidden, desc.out_dim, desc.samples, desc.data_seed)
        if key not in self._objs:
            self._objs[key] = self.lib.orc_objective_create(desc.kind, desc.in_dim, desc.hidden,
                                                            desc.out_dim, desc.samples, desc.data_seed)
        return self._objs[key]

    def dataset(self, desc: ObjectiveDesc):
        h = self.objective(desc)
        I = 784 if desc.kind == OBJ_LENET else desc.in_dim
        X = np.ctypeslib.as_array(self.lib.orc_objective_data(h), shape=(desc.samples * I,)).copy()
        y = np.ctypeslib.as_array(self.lib.orc_objective_labels(h), shape=(desc.samples,)).copy()
        return X.reshape(desc.samples, I), y

    def evaluate(self, desc: ObjectiveDesc, x) -> float:
        x = _arr(x)
        return float(self.lib.orc_objective_eval(self.objective(desc), _p(x), x.size))

    def batched_apply(self, desc: ObjectiveDesc, rows) -> tuple[np.ndarray, int]:
        rows = _arr(rows)
        n, d = rows.shape[-2] if rows.ndim == 3 else rows.shape[0], rows.shape[-1]
        flat = rows.reshape(-1, d)
        out = np.empty(flat.shape[0])
        nan = self.lib.orc_batched_apply(self.objective(desc), _p(flat), flat.shape[0], d, _p(out))
        return out.reshape(rows.shape[:-1]), int(nan)

    def argmin_per_population(self, fitness):
        f = _arr(fitness)
        idx = np.empty(f.shape[0], dtype=np.uint64)
        val = np.empty(f.shape[0])
        self.lib.orc_argmin_per_population(_p(f), f.shape[0], f.shape[1],
                                           idx.ctypes.data_as(_pu64), _p(val))
        return idx, val

    # -- engine operators (array shapes follow BatchCube [B][N][D])
    def initialize_positions(self, cfg: Config, lower, upper, seed):
        lo, hi = _arr(lower), _arr(upper)
        c, keep = _cconfig(cfg)
        out = np.empty((cfg.batches, cfg.fireworks, lo.size))
        self.lib.orc_initialize_positions(C.byref(c), _p(lo), _p(hi), lo.size, seed, _p(out))
        return out

    def population_range(self, pos):
        pos = _arr(pos)
        B, mu, D = pos.shape
        lo, hi = np.empty((B, D)), np.empty((B, D))
        self.lib.orc_population_range(_p(pos), B, mu, D, _p(lo), _p(hi))
        return lo, hi

    def explode(self, pos, amp, lam, iteration, seed):
        pos, amp = _arr(pos), _arr(amp)
        B, mu, D = pos.shape
        out = np.empty((B, mu * lam, D))
        self.lib.orc_explode(_p(pos), _p(amp), B, mu, D, lam, iteration, seed, _p(out))
        return out

    def random_mapping(self, cand, per, pos, lower, upper, iteration, seed, stream):
        cand, pos = _arr(cand).copy(), _arr(pos)
        lo, hi = _arr(lower), _arr(upper)
        B, rows, D = cand.shape
        self.lib.orc_random_mapping(_p(cand), B, rows, D, per, _p(pos), pos.shape[1], _p(lo), _p(hi),
                                    iteration, seed, stream)
        return cand

    def guiding_vector(self, sparks, spark_fit, lam, top):
        s, f = _arr(sparks), _arr(spark_fit)
        B, rows, D = s.shape
        mu = rows // lam
        out = np.empty((B, mu, D))
        r = self.lib.orc_guiding_vector(_p(s), _p(f), B, mu, lam, D, top, _p(out))
        if r != 0:
            raise ValueError("guiding_vector: elite and poor sets overlap")
        return out

    def multi_guiding_sparks(self, pos, delta, boosts):
        pos, dl, bt = _arr(pos), _arr(delta), _arr(boosts)
        B, mu, D = pos.shape
        out = np.empty((B, mu * bt.size, D))
        self.lib.orc_multi_guiding_sparks(_p(pos), _p(dl), B, mu, D, _p(bt), bt.size, _p(out))
        return out

    def select_best(self, pos, fit, sparks, spark_fit, lam, guides=None, guide_fit=None, M=0):
        pos, fit, s, sf = _arr(pos), _arr(fit), _arr(sparks), _arr(spark_fit)
        B, mu, D = pos.shape
        npos, nfit, nli, imp = np.empty_like(pos), np.empty((B, mu)), np.empty((B, mu)), np.empty((B, mu))
        if guides is not None:
            g, gf = _arr(guides), _arr(guide_fit)
            gp, gfp = _p(g), _p(gf)
        else:
            gp, gfp, M = None, None, 0
        self.lib.orc_select_best(_p(pos), _p(fit), B, mu, D, _p(s), _p(sf), lam, gp, gfp, M,
                                 _p(npos), _p(nfit), _p(nli), _p(imp))
        return npos, nfit, nli, imp

    def update_amplitudes(self, amp, improved, amp_amplify, amp_reduce, max_range):
        a, im = _arr(amp), _arr(improved)
        out = np.empty_like(a)
        self.lib.orc_update_amplitudes(_p(a), _p(im), a.size, amp_amplify, amp_reduce, max_range, _p(out))
        return out

    def loser_out(self, pos, fit, amp, li, cfg: Config, lower, upper, iteration, seed, iters_rem,
                  desc: ObjectiveDesc):
        pos, fit, amp, li = (_arr(x).copy() for x in (pos, fit, amp, li))
        lo, hi = _arr(lower), _arr(upper)
        B, mu, D = pos.shape
        c, keep = _cconfig(cfg)
        nan = C.c_uint64(0)
        n = self.lib.orc_loser_out(_p(pos), _p(fit), _p(amp), _p(li), B, mu, D, C.byref(c), _p(lo), _p(hi),
                                   iteration, seed, iters_rem, self.objective(desc), C.byref(nan))
        return pos, fit, amp, li, int(n)

    def run(self, cfg: Config, lower, upper, desc: ObjectiveDesc, seed: int) -> Record:
        lo, hi = _arr(lower), _arr(upper)
        D = lo.size
        c, keep = _cconfig(cfg)
        cap = _trace_cap(cfg)
        B = cfg.batches
        bf, bp = np.empty(B), np.zeros((B, D))
        te, tb, tw = np.zeros((B, cap), dtype=np.uint64), np.zeros((B, cap)), np.zeros((B, cap))
        cnt = _Counters()
        err = self.lib.orc_run(C.byref(c), _p(lo), _p(hi), D, self.objective(desc), seed, _p(bf), _p(bp),
                               te.ctypes.data_as(_pu64), _p(tb), _p(tw), cap, C.byref(cnt))
        if err is not None:
            raise ValueError(err.decode())
        w = int(cnt.waves)
        return Record(bf, bp, te[:, :w], tb[:, :w], tw[:, :w], int(cnt.evaluations_used),
                      int(cnt.iterations), int(cnt.losers_reinitialized), int(cnt.nan_evaluations))


class Reference:
    """ctypes wrapper of the compiled reference (oracle/_ref/libmgfwa_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_key_hash.restype = _u64
        L.ref_key_hash.argtypes = [_u64] * 7
        L.ref_uniform_sample.restype = C.c_int
        L.ref_uniform_sample.argtypes = [_u64] * 7 + [_dbl, _dbl, _pd]
        L.ref_config_validate.argtypes = [C.POINTER(_CConfig), C.c_char_p, C.c_size_t]
        L.ref_top_spark_count.restype = _u64
        L.ref_objective_eval.restype = _dbl
        L.ref_objective_eval.argtypes = [C.POINTER(_CObjDesc), _pd, _u64]
        L.ref_batched_apply.argtypes = [C.POINTER(_CObjDesc), _pd, _u64, _u64, _u64, C.c_int, _pd, _pu64]
        L.ref_argmin_per_population.argtypes = [_pd, _u64, _u64, _pu64, _pd]
        L.ref_initialize.argtypes = [C.POINTER(_CConfig), _pd, _pd, _u64, C.POINTER(_CObjDesc), C.c_int, _u64,
                                     _pd, _pd, _pd, C.c_char_p, C.c_size_t]
        L.ref_explode.argtypes = [_pd, _pd, _u64, _u64, _u64, C.POINTER(_CConfig), _u64, _u64, _pd]
        L.ref_random_mapping.argtypes = [_pd, _u64, _u64, _u64, _u64, _pd, _u64, _pd, _pd, _u64, _u64, _u64, _pd]
        L.ref_guiding_vector.argtypes = [_pd, _pd, _u64, _u64, _u64, C.POINTER(_CConfig), _pd, C.c_char_p,
                                         C.c_size_t]
        L.ref_multi_guiding_sparks.argtypes = [_pd, _pd, _u64, _u64, _u64, C.POINTER(_CConfig), _pd]
        L.ref_select_best.argtypes = [_pd, _pd, _u64, _u64, _u64, _pd, _pd, _u64, _pd, _pd, _u64, _pd, _pd, _pd,
                                      _pd]
        L.ref_update_amplitudes.argtypes = [_pd, _pd, _u64, _u64, C.POINTER(_CConfig), _dbl, _pd]
        L.ref_loser_out.argtypes = [_pd, _pd, _pd, _pd, _pu64, _u64, _u64, _u64, C.POINTER(_CConfig), _pd, _pd,
                                    _u64, _u64, _dbl, C.POINTER(_CObjDesc), C.c_int, _pu64]
        L.ref_run.argtypes = [C.POINTER(_CConfig), _pd, _pd, _u64, C.POINTER(_CObjDesc), C.c_int, _u64, _pd, _pd,
                              _pu64, _pd, _pd, _u64, C.POINTER(_Counters), C.c_char_p, C.c_size_t]

    def key_hash(self, seed, stream, it, b, n, k, d) -> int:
        return int(self.lib.ref_key_hash(seed, stream, it, b, n, k, d))

    def uniform_sample(self, seed, stream, it, b, n, k, d, lo, hi) -> float:
        out = C.c_double()
        if self.lib.ref_uniform_sample(seed, stream, it, b, n, k, d, lo, hi, C.byref(out)) != 0:
            raise ValueError("uniform_sample: lo must be <= hi")
        return out.value

    def validate(self, cfg: Config) -> Optional[str]:
        c, keep = _cconfig(cfg)
        buf = C.create_string_buffer(512)
        r = self.lib.ref_config_validate(C.byref(c), buf, 512)
        return None if r == 0 else buf.value.decode()

    def evaluate(self, desc: ObjectiveDesc, x) -> float:
        x = _arr(x)
        d = _cobj(desc)
        return float(self.lib.ref_objective_eval(C.byref(d), _p(x), x.size))

    def batched_apply(self, desc: ObjectiveDesc, rows, workers: int = 0):
        rows = _arr(rows)
        B, N, D = rows.shape
        out = np.empty((B, N))
        nan = C.c_uint64(0)
        d = _cobj(desc)
        r = self.lib.ref_batched_apply(C.byref(d), _p(rows), B, N, D, workers, _p(out), C.byref(nan))
        if r != 0:
            raise ValueError("batched_apply failed")
        return out, int(nan.value)

    def argmin_per_population(self, fitness):
        f = _arr(fitness)
        idx = np.empty(f.shape[0], dtype=np.uint64)
        val = np.empty(f.shape[0])
        self.lib.ref_argmin_per_population(_p(f), f.shape[0], f.shape[1], idx.ctypes.data_as(_pu64), _p(val))
        return idx, val

    def initialize(self, cfg: Config, lower, upper, desc: ObjectiveDesc, seed, workers=0):
        lo, hi = _arr(lower), _arr(upper)
        c, keep = _cconfig(cfg)
        d = _cobj(desc)
        pos = np.empty((cfg.batches, cfg.fireworks, lo.size))
        fit, amp = np.empty((cfg.batches, cfg.fireworks)), np.empty((cfg.batches, cfg.fireworks))
        buf = C.create_string_buffer(512)
        if self.lib.ref_initialize(C.byref(c), _p(lo), _p(hi), lo.size, C.byref(d), workers, seed, _p(pos),
                                   _p(fit), _p(amp), buf, 512) != 0:
            raise ValueError(buf.value.decode())
        return pos, fit, amp

    def explode(self, pos, amp, cfg: Config, iteration, seed):
        pos, amp = _arr(pos), _arr(amp)
        B, mu, D = pos.shape
        c, keep = _cconfig(cfg)
        out = np.empty((B, mu * cfg.sparks_per_firework, D))
        self.lib.ref_explode(_p(pos), _p(amp), B, mu, D, C.byref(c), iteration, seed, _p(out))
        return out

    def random_mapping(self, cand, per, pos, lower, upper, iteration, seed, stream):
        cand, pos, lo, hi = _arr(cand), _arr(pos), _arr(lower), _arr(upper)
        B, rows, D = cand.shape
        out = np.empty_like(cand)
        self.lib.ref_random_mapping(_p(cand), B, rows, D, per, _p(pos), pos.shape[1], _p(lo), _p(hi), iteration,
                                    seed, stream, _p(out))
        return out

    def guiding_vector(self, sparks, spark_fit, cfg: Config):
        s, f = _arr(sparks), _arr(spark_fit)
        B, rows, D = s.shape
        mu = rows // cfg.sparks_per_firework
        c, keep = _cconfig(cfg)
        out = np.empty((B, mu, D))
        buf = C.create_string_buffer(512)
        if self.lib.ref_guiding_vector(_p(s), _p(f), B, mu, D, C.byref(c), _p(out), buf, 512) != 0:
            raise ValueError(buf.value.decode())
        return out

    def multi_guiding_sparks(self, pos, delta, cfg: Config):
        pos, dl = _arr(pos), _arr(delta)
        B, mu, D = pos.shape
        c, keep = _cconfig(cfg)
        out = np.empty((B, mu * cfg.guides_per_firework, D))
        self.lib.ref_multi_guiding_sparks(_p(pos), _p(dl), B, mu, D, C.byref(c), _p(out))
        return out

    def select_best(self, pos, fit, sparks, spark_fit, lam, guides=None, guide_fit=None, M=0):
        pos, fit, s, sf = _arr(pos), _arr(fit), _arr(sparks), _arr(spark_fit)
        B, mu, D = pos.shape
        npos, nfit, nli, imp = np.empty_like(pos), np.empty((B, mu)), np.empty((B, mu)), np.empty((B, mu))
        if guides is not None:
            g, gf = _arr(guides), _arr(guide_fit)
            gp, gfp = _p(g), _p(gf)
        else:
            gp, gfp, M = None, None, 0
        self.lib.ref_select_best(_p(pos), _p(fit), B, mu, D, _p(s), _p(sf), lam, gp, gfp, M, _p(npos), _p(nfit),
                                 _p(nli), _p(imp))
        return npos, nfit, nli, imp

    def update_amplitudes(self, amp, improved, cfg: Config, max_range):
        a, im = _arr(amp), _arr(improved)
        c, keep = _cconfig(cfg)
        out = np.empty_like(a)
        a2 = a.reshape(a.shape[0], -1) if a.ndim > 1 else a.reshape(1, -1)
        self.lib.ref_update_amplitudes(_p(a), _p(im), a2.shape[0], a2.shape[1], C.byref(c), max_range, _p(out))
        return out

    def loser_out(self, pos, fit, amp, li, used, cfg: Config, lower, upper, iteration, seed, iters_rem,
                  desc: ObjectiveDesc, workers=0):
        pos, fit, amp, li = (_arr(x).copy() for x in (pos, fit, amp, li))
        lo, hi = _arr(lower), _arr(upper)
        B, mu, D = pos.shape
        c, keep = _cconfig(cfg)
        d = _cobj(desc)
        u = C.c_uint64(used)
        n = C.c_uint64(0)
        self.lib.ref_loser_out(_p(pos), _p(fit), _p(amp), _p(li), C.byref(u), B, mu, D, C.byref(c), _p(lo), _p(hi),
                               iteration, seed, iters_rem, C.byref(d), workers, C.byref(n))
        return pos, fit, amp, li, int(n.value), int(u.value)

    def run(self, cfg: Config, lower, upper, desc: ObjectiveDesc, seed: int, workers: int = 0) -> Record:
        lo, hi = _arr(lower), _arr(upper)
        D = lo.size
        c, keep = _cconfig(cfg)
        d = _cobj(desc)
        cap = _trace_cap(cfg)
        B = cfg.batches
        bf, bp = np.empty(B), np.zeros((B, D))
        te, tb, tw = np.zeros((B, cap), dtype=np.uint64), np.zeros((B, cap)), np.zeros((B, cap))
        cnt = _Counters()
        buf = C.create_string_buffer(512)
        r = self.lib.ref_run(C.byref(c), _p(lo), _p(hi), D, C.byref(d), workers, seed, _p(bf), _p(bp),
                             te.ctypes.data_as(_pu64), _p(tb), _p(tw), cap, C.byref(cnt), buf, 512)
        if r != 0:
            raise ValueError(buf.value.decode())
        w = int(cnt.waves)
        return Record(bf, bp, te[:, :w], tb[:, :w], tw[:, :w], int(cnt.evaluations_used), int(cnt.iterations),
                      int(cnt.losers_reinitialized), int(cnt.nan_evaluations))
