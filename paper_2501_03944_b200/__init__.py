"""paper_2501_03944_b200 — B200-native GPU-MGFWA generation engine.

The hot path (one MGFWA generation: explosion sparks, fitness, guiding
sparks, selection, amplitude adaptation, loser-out) runs as hand-written
sm_100a CUDA kernels in ``libmgfwa_b200.so``; this package is the Python
mirror of the reference's C++ optimizer / objective interface over that
library's C-ABI (include/mgfwa_b200.h).
"""
from .engine import (  # noqa: F401
    Ackley,
    CandidateSet,
    CudaError,
    Engine,
    FireworkState,
    LeNet,
    MgfwaConfig,
    MlpWeights,
    NET_REGISTRY,
    Net,
    Objective,
    Rastrigin,
    RunRecord,
    SearchSpace,
    SelectionResult,
    Sphere,
    argmin_per_population,
    batched_apply,
    explode,
    explode_map,
    guides_map,
    guiding_vector,
    initialize,
    kExplode,
    kGuide,
    kInit,
    kMapping,
    kReinit,
    key_hash,
    loser_out,
    net_param_count,
    multi_guiding_sparks,
    random_mapping,
    run,
    select_best,
    update_amplitudes,
)

__version__ = "0.1.0"
