"""ctypes binding of include/mgfwa_b200.h (the library's C-ABI).

Loads the in-tree ``libmgfwa_b200.so``; there is no fallback: if the CUDA
library is missing the import fails loudly (build it with
``python -m paper_2501_03944_b200.build``).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MGFWA_LIB: an alternative build of the same library (A/B experiments,
# scripts/build_variant.py); the in-tree build is the default.
LIB_PATH = os.environ.get("MGFWA_LIB") or os.path.join(HERE, "libmgfwa_b200.so")

MGFWA_OK, MGFWA_EINVAL, MGFWA_ECUDA, MGFWA_ENOMEM, MGFWA_ENCCL, MGFWA_ESTATE = range(6)
OBJ_SPHERE, OBJ_RASTRIGIN, OBJ_ACKLEY, OBJ_MLP_WEIGHTS, OBJ_LENET, OBJ_NET = 1, 2, 3, 4, 5, 6

_u64, _dbl, _int = C.c_uint64, C.c_double, C.c_int
_pd, _pu64 = C.POINTER(C.c_double), C.POINTER(C.c_uint64)


class mgfwa_config_t(C.Structure):
    _fields_ = [("batches", _u64), ("fireworks", _u64), ("sparks_per_firework", _u64),
                ("guides_per_firework", _u64), ("guide_fraction", _dbl), ("boosts", _pd),
                ("n_boosts", _u64), ("amp_amplify", _dbl), ("amp_reduce", _dbl),
                ("initial_amplitude", _dbl), ("max_evaluations", _u64),
                ("wall_clock_budget_ms", _dbl)]


class mgfwa_space_t(C.Structure):
    _fields_ = [("lower", _pd), ("upper", _pd), ("dim", _u64)]


class mgfwa_objective_t(C.Structure):
    _fields_ = [("kind", _int), ("in_dim", C.c_uint32), ("hidden", C.c_uint32),
                ("out_dim", C.c_uint32), ("samples", C.c_uint32), ("data_seed", _u64),
                ("net_id", _int), ("weight_seed", _u64)]


class mgfwa_counters_t(C.Structure):
    _fields_ = [("evaluations_used", _u64), ("iterations", _u64),
                ("losers_reinitialized", _u64), ("nan_evaluations", _u64),
                ("trace_waves", _u64)]


_P = C.c_void_p
# name -> (restype, argtypes); mirrors include/mgfwa_b200.h one to one.
SIGNATURES = {
    "mgfwa_version": (C.c_char_p, []),
    "mgfwa_release_cached_workspace": (_int, []),
    "mgfwa_last_error": (C.c_char_p, [_P]),
    "mgfwa_create": (_int, [C.POINTER(mgfwa_config_t), C.POINTER(mgfwa_space_t),
                            C.POINTER(mgfwa_objective_t), _u64, _int, C.POINTER(_P)]),
    "mgfwa_destroy": (_int, [_P]),
    "mgfwa_set_stream": (_int, [_P, _P]),
    "mgfwa_kernels_per_generation": (_int, [_P, _pu64]),
    "mgfwa_initialize": (_int, [_P]),
    "mgfwa_step": (_int, [_P, _u64, _pu64]),
    "mgfwa_enqueue_generations": (_int, [_P, _u64]),
    "mgfwa_sync": (_int, [_P]),
    "mgfwa_run": (_int, [_P, C.POINTER(mgfwa_counters_t)]),
    "mgfwa_get_counters": (_int, [_P, C.POINTER(mgfwa_counters_t)]),
    "mgfwa_get_best": (_int, [_P, _pd, _pd]),
    "mgfwa_get_trace": (_int, [_P, _pu64, _pd, _pd, _u64, _pu64]),
    "mgfwa_get_state": (_int, [_P, _pd, _pd, _pd, _pd]),
    "mgfwa_get_candidates": (_int, [_P, _pd, _pd, _pd, _pd, C.POINTER(C.c_uint16)]),
    "mgfwa_run_once": (_int, [C.POINTER(mgfwa_config_t), C.POINTER(mgfwa_space_t),
                              C.POINTER(mgfwa_objective_t), _u64, _int, _pd, _pd, _pu64, _pd, _pd,
                              _u64, C.POINTER(mgfwa_counters_t)]),
    "mgfwa_op_initialize": (_int, [C.POINTER(mgfwa_config_t), C.POINTER(mgfwa_space_t),
                                   C.POINTER(mgfwa_objective_t), _u64, _pd, _pd, _pd]),
    "mgfwa_op_explode_map": (_int, [C.POINTER(mgfwa_config_t), C.POINTER(mgfwa_space_t), _pd, _pd,
                                    _u64, _u64, _pd]),
    "mgfwa_op_random_mapping": (_int, [C.POINTER(mgfwa_space_t), _pd, _u64, _u64, _u64, _pd, _u64,
                                       _u64, _u64, _u64, _pd]),
    "mgfwa_op_guiding_vector": (_int, [C.POINTER(mgfwa_config_t), _u64, _pd, _pd, _pd]),
    "mgfwa_op_guides": (_int, [C.POINTER(mgfwa_config_t), C.POINTER(mgfwa_space_t), _pd, _pd, _pd,
                               _u64, _u64, _pd]),
    "mgfwa_op_select_best": (_int, [C.POINTER(mgfwa_config_t), C.POINTER(mgfwa_space_t), _pd, _pd,
                                    _pd, _pd, _pd, _pd, _pd, _pd, _pd, _pd, _pd, _pd]),
    "mgfwa_op_loser_out": (_int, [C.POINTER(mgfwa_config_t), C.POINTER(mgfwa_space_t),
                                  C.POINTER(mgfwa_objective_t), _pd, _pd, _pd, _pd, _pu64, _u64,
                                  _u64, _dbl, _pu64]),
    "mgfwa_op_batched_apply": (_int, [C.POINTER(mgfwa_objective_t), _pd, _u64, _u64, _pd, _pu64]),
    "mgfwa_op_argmin_per_population": (_int, [_pd, _u64, _u64, _pu64, _pd]),
    "mgfwa_key_hash": (_int, [_pu64, _u64, _pu64]),
    "mgfwa_validate_config": (_int, [C.POINTER(mgfwa_config_t)]),
    "mgfwa_time_fitness": (_int, [_P, _u64, _pd, _pu64]),
    "mgfwa_time_kernel": (_int, [_P, _int, _u64, _pd, _pu64]),
    "mgfwa_create_shard": (_int, [C.POINTER(mgfwa_config_t), C.POINTER(mgfwa_space_t),
                                  C.POINTER(mgfwa_objective_t), _u64, _int, _int, _int, C.POINTER(_P)]),
    "mgfwa_nccl_unique_id": (_int, [_P]),
    "mgfwa_attach_nccl": (_int, [_P, _P, _int, _int]),
    "mgfwa_generation_phase": (_int, [_P, _int]),
    "mgfwa_shard_exchange": (_int, [_P, _P]),
    "mgfwa_set_shard_mode": (_int, [_P, _int]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded CUDA library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA library with "
                "`python -m paper_2501_03944_b200.build` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
