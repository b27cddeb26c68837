/*
 * mgfwa_b200.h — C-ABI of the B200-native MGFWA generation engine.
 *
 * This is the drop-in boundary for the reference's generation loop.  Every
 * entry point names the reference interface it replaces (paths relative to
 * /root/reference/proj).  Plain pointers and sizes only; no CUDA or torch
 * types cross this boundary (a cudaStream_t may be passed as void*).
 *
 * Status codes: MGFWA_OK (0) or one of MGFWA_E*; the message of the last
 * failure is available from mgfwa_last_error().  MGFWA_EINVAL carries the
 * reference's std::invalid_argument message verbatim where one exists
 * (config.cpp:26-77, engine.cpp:136-141, 321-323, backend.cpp:30-35).
 *
 * There is no host callback, no CPU fallback and no multi-backend dispatch:
 * the objective is a closed descriptor evaluated on the GPU.
 */
#ifndef MGFWA_B200_H
#define MGFWA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGFWA_OK 0
#define MGFWA_EINVAL 1 /* std::invalid_argument in the reference   */
#define MGFWA_ECUDA 2  /* CUDA runtime / driver failure             */
#define MGFWA_ENOMEM 3 /* device or host allocation failure         */
#define MGFWA_ENCCL 4  /* collective failure (sharded runs)         */
#define MGFWA_ESTATE 5 /* call out of order (e.g. step before init) */

/* MgfwaConfig, config.hpp:33-47, field by field (boosts as pointer + M). */
typedef struct {
  uint64_t batches;             /* B                               */
  uint64_t fireworks;           /* mu                              */
  uint64_t sparks_per_firework; /* lambda                          */
  uint64_t guides_per_firework; /* M; 0 disables guiding sparks    */
  double guide_fraction;        /* sigma in (0, 0.5]               */
  const double* boosts;         /* beta_1..beta_M, beta_1 = 1      */
  uint64_t n_boosts;
  double amp_amplify;           /* C_a > 1                         */
  double amp_reduce;            /* C_r in (0, 1)                   */
  double initial_amplitude;     /* A_0; <= 0 means 0.5 * max range */
  uint64_t max_evaluations;     /* 0 = unlimited                   */
  double wall_clock_budget_ms;  /* 0 = unlimited                   */
} mgfwa_config_t;

/* SearchSpace, config.hpp:11-28. */
typedef struct {
  const double* lower;
  const double* upper;
  uint64_t dim;
} mgfwa_space_t;

/* Objective descriptor replacing the std::function Objective of
 * backend.hpp:15 (a host callback cannot run on the device). */
#define MGFWA_OBJ_SPHERE 1      /* nets.cpp:80-84                          */
#define MGFWA_OBJ_RASTRIGIN 2   /* 10 D + sum(x^2 - 10 cos 2 pi x)          */
#define MGFWA_OBJ_ACKLEY 3      /* standard Ackley, unshifted               */
#define MGFWA_OBJ_MLP_WEIGHTS 4 /* mean CE of an I-H-O ReLU MLP whose
                                   weights are the candidate (tensor cores) */
#define MGFWA_OBJ_LENET 5       /* mean CE of LeNet-5 whose 61,706 parameters
                                   are the candidate (28x28 samples)       */
#define MGFWA_OBJ_NET 6         /* the reference's input-space benchmark
                                   network net_id (nets.cpp:36-167): fixed
                                   weights from weight_seed, the candidate
                                   is the input vector; fp64 on the device */
typedef struct {
  int kind;
  uint32_t in_dim;   /* MLP: I (e.g. 784)            */
  uint32_t hidden;   /* MLP: H (32, 64, 128, 256)    */
  uint32_t out_dim;  /* MLP: O (<= 10)               */
  uint32_t samples;  /* MLP / LeNet: S synthetic samples */
  uint64_t data_seed;
  int net_id;            /* NET: 1..12 (net_registry, nets.cpp:36-55) */
  uint64_t weight_seed;  /* NET: MlpBlackBox weight seed             */
} mgfwa_objective_t;

/* RunRecord counters, engine.hpp:63-66. */
typedef struct {
  uint64_t evaluations_used;
  uint64_t iterations;
  uint64_t losers_reinitialized;
  uint64_t nan_evaluations;
  uint64_t trace_waves; /* trace points per batch so far */
} mgfwa_counters_t;

typedef struct mgfwa_ctx* mgfwa_ctx_t;

/* ---- context lifecycle ------------------------------------------------ */
/* Validates (MgfwaConfig::validate config.cpp:42-79, SearchSpace::validate
 * config.cpp:25-35, the budget check engine.cpp:319-323) and allocates all
 * device state on `device`.  Inputs are copied (value semantics). */
int mgfwa_create(const mgfwa_config_t* config, const mgfwa_space_t* space,
                 const mgfwa_objective_t* objective, uint64_t seed, int device,
                 mgfwa_ctx_t* out);
int mgfwa_destroy(mgfwa_ctx_t ctx);
/* Message of the last failure on ctx (or of the last failed call without
 * a ctx when ctx == NULL). */
const char* mgfwa_last_error(mgfwa_ctx_t ctx);
/* Run subsequent work on an external stream (cudaStream_t as void*). */
int mgfwa_set_stream(mgfwa_ctx_t ctx, void* cuda_stream);
/* Number of graph-replayed kernels one generation launches; 0 when the
 * context runs the persistent small-problem loop (analytic objective,
 * D <= 512, one context), which executes any number of generations in one
 * kernel launch per enqueue. */
int mgfwa_kernels_per_generation(mgfwa_ctx_t ctx, uint64_t* n);

/* ---- the generation loop (engine.hpp:71-132) --------------------------- */
/* initialize(), engine.cpp:45-76, plus record_wave #0 (engine.cpp:353). */
int mgfwa_initialize(mgfwa_ctx_t ctx);
/* Up to max_generations loop bodies (engine.cpp:359-417), stopping at the
 * budget; *generations_run receives the count.  Synchronous. */
int mgfwa_step(mgfwa_ctx_t ctx, uint64_t max_generations,
               uint64_t* generations_run);
/* Asynchronous: enqueue n loop bodies (one CUDA-graph replay each) on the
 * context stream and return.  Generations past the budget are no-ops on
 * the device.  Follow with mgfwa_sync(). */
int mgfwa_enqueue_generations(mgfwa_ctx_t ctx, uint64_t n);
int mgfwa_sync(mgfwa_ctx_t ctx);
/* run(), engine.cpp:313-423: initialize, then loop to the budget. */
int mgfwa_run(mgfwa_ctx_t ctx, mgfwa_counters_t* counters);

/* ---- results (RunRecord, engine.hpp:56-67) ----------------------------- */
int mgfwa_get_counters(mgfwa_ctx_t ctx, mgfwa_counters_t* out);
/* best_fitness[B], best_position[B][D] */
int mgfwa_get_best(mgfwa_ctx_t ctx, double* best_fitness,
                   double* best_position);
/* trace arrays [B][cap]; *waves = trace points per batch (may exceed cap:
 * only the first cap are written). */
int mgfwa_get_trace(mgfwa_ctx_t ctx, uint64_t* evaluations, double* best,
                    double* wall_ms, uint64_t cap, uint64_t* waves);
/* FireworkState, engine.hpp:16-22: pos[B][mu][D], fit/amp/li[B][mu] */
int mgfwa_get_state(mgfwa_ctx_t ctx, double* positions, double* fitness,
                    double* amplitudes, double* last_improvement);

/* The candidate sets of the last generation run on ctx, as the reference's
 * run() loop holds them before select_best (engine.cpp:369-384): the mapped
 * sparks [Fl*lambda][D] (SparkSet.positions after random_mapping, kMapping)
 * with their fitness, the mapped guiding sparks [Fl*M][D] (GuideSet after
 * random_mapping, kGuide) with their fitness, and, for the tensor-core
 * objectives, the bf16 shadow of the sparks the fitness kernel read.  Fl =
 * fireworks owned by ctx (B*mu unsharded).  Any pointer may be NULL.  Used by
 * the parity tests to check the real generation path step by step. */
int mgfwa_get_candidates(mgfwa_ctx_t ctx, double* sparks, double* spark_fitness,
                         double* guides, double* guide_fitness,
                         uint16_t* sparks_bf16);

/* One-shot run() over host buffers — the plain drop-in for
 * run(config, space, objective, backend, seed) (engine.hpp:130-132).
 * trace arrays are [B][trace_cap] and may be NULL. */
int mgfwa_run_once(const mgfwa_config_t* config, const mgfwa_space_t* space,
                   const mgfwa_objective_t* objective, uint64_t seed,
                   int device, double* best_fitness, double* best_position,
                   uint64_t* trace_evaluations, double* trace_best,
                   double* trace_wall_ms, uint64_t trace_cap,
                   mgfwa_counters_t* counters);

/* ---- operator seams on host arrays (engine.hpp:71-125) ----------------
 * They run the same device kernels the generation loop runs.  Host arrays
 * are fp64 in the reference layout (BatchCube [B][N][D] row-major); device
 * state is fp32 (positions) / fp64 (amplitudes, fitness). */
/* initialize(), engine.cpp:45-76: pos[B][mu][D], fit[B][mu], amp[B][mu] */
int mgfwa_op_initialize(const mgfwa_config_t* config,
                        const mgfwa_space_t* space,
                        const mgfwa_objective_t* objective, uint64_t seed,
                        double* positions, double* fitness,
                        double* amplitudes);
/* random_mapping(explode(...), kMapping), engine.cpp:78-131, fused. */
int mgfwa_op_explode_map(const mgfwa_config_t* config,
                         const mgfwa_space_t* space, const double* positions,
                         const double* amplitudes, uint64_t iteration,
                         uint64_t seed, double* sparks);
/* random_mapping, engine.cpp:103-131: cand[B][rows][D], pos[B][mu][D] */
int mgfwa_op_random_mapping(const mgfwa_space_t* space, const double* cand,
                            uint64_t B, uint64_t rows, uint64_t per,
                            const double* positions, uint64_t mu,
                            uint64_t iteration, uint64_t seed,
                            uint64_t stream, double* out);
/* guiding_vector, engine.cpp:133-172: delta[B][mu][D] (fp32-rounded). */
int mgfwa_op_guiding_vector(const mgfwa_config_t* config, uint64_t dim,
                            const double* sparks, const double* spark_fitness,
                            double* delta);
/* random_mapping(multi_guiding_sparks(guiding_vector(...)), kGuide),
 * engine.cpp:133-196, fused: guides[B][mu*M][D]. */
int mgfwa_op_guides(const mgfwa_config_t* config, const mgfwa_space_t* space,
                    const double* positions, const double* sparks,
                    const double* spark_fitness, uint64_t iteration,
                    uint64_t seed, double* guides);
/* select_best + update_amplitudes, engine.cpp:198-256.  guides may be NULL
 * when M = 0.  Outputs: new pos/fit/li/amp, improved (0/1 as double). */
int mgfwa_op_select_best(const mgfwa_config_t* config,
                         const mgfwa_space_t* space, const double* positions,
                         const double* fitness, const double* amplitudes,
                         const double* sparks, const double* spark_fitness,
                         const double* guides, const double* guide_fitness,
                         double* new_positions, double* new_fitness,
                         double* new_last_improvement, double* improved,
                         double* new_amplitudes);
/* loser_out, engine.cpp:258-311, in place on pos/fit/amp/li; returns the
 * number of reinitialized fireworks in *reinit and adds it to *used. */
int mgfwa_op_loser_out(const mgfwa_config_t* config,
                       const mgfwa_space_t* space,
                       const mgfwa_objective_t* objective, double* positions,
                       double* fitness, double* amplitudes,
                       double* last_improvement, uint64_t* used,
                       uint64_t iteration, uint64_t seed,
                       double iterations_remaining, uint64_t* reinit);
/* batched_apply, backend.cpp:28-67: fitness[N] of rows[N][D]; NaN -> +inf
 * counted in *nan_count. */
int mgfwa_op_batched_apply(const mgfwa_objective_t* objective,
                           const double* rows, uint64_t n, uint64_t dim,
                           double* fitness, uint64_t* nan_count);
/* argmin_per_population, backend.cpp:69-83 */
int mgfwa_op_argmin_per_population(const double* fitness, uint64_t rows,
                                   uint64_t cols, uint64_t* index,
                                   double* value);

/* ---- firework sharding across GPUs ---------------------
 * The B*mu fireworks are split into `world` equal contiguous shards; rank r
 * explodes, evaluates, guides and selects fireworks [r*F/world, (r+1)*F/world)
 * and keeps a replica of every firework's {position, fitness, amplitude,
 * last improvement}, refreshed once per generation by an in-place NCCL
 * all-gather (NVLink).  Population range, loser-out (all losers are re-drawn
 * from kReinit and evaluated by every rank) and record_wave then run
 * identically on all ranks, so a sharded run is bit-identical to the
 * single-GPU run.  Requires F % world == 0 and an evaluation budget (no
 * wall-clock budget: every rank must take the same termination decision). */
int mgfwa_create_shard(const mgfwa_config_t* config, const mgfwa_space_t* space,
                       const mgfwa_objective_t* objective, uint64_t seed,
                       int device, int rank, int world, mgfwa_ctx_t* out);
/* 128-byte ncclUniqueId (created on rank 0, broadcast by the caller). */
int mgfwa_nccl_unique_id(void* out128);
int mgfwa_attach_nccl(mgfwa_ctx_t ctx, const void* unique_id128, int nranks,
                      int rank);
/* Shard modes (before mgfwa_initialize).  MGFWA_SHARD_FIREWORK (default):
 * as above.  MGFWA_SHARD_REPLICA (needs batches % world == 0): each rank
 * owns whole batches — replicas of the optimisation, SURVEY.md §8(f) rank 4 —
 * and runs loser-out, record_wave and the population range for its own
 * batches only; batches interact only through the shared evaluation budget
 * (loser-out adds every batch's losers, engine.cpp:309), so the
 * per-generation exchange is a single 8-byte NCCL all-reduce of the loser
 * count.  Results (trace, best, state) are valid for the rank's own batches;
 * trace entries of other batches read NaN.  Counters are global. */
#define MGFWA_SHARD_FIREWORK 0
#define MGFWA_SHARD_REPLICA 1
int mgfwa_set_shard_mode(mgfwa_ctx_t ctx, int mode);
/* Manual stepping without NCCL (tests, one-process emulation): phase 1 =
 * pop range .. selection, phase 2 = loser-out .. record_wave; between them
 * every shard imports every other shard's owned rows (replica mode: adds
 * their loser counts; phase 1 then ends with loser-out). */
int mgfwa_generation_phase(mgfwa_ctx_t ctx, int phase);
int mgfwa_shard_exchange(mgfwa_ctx_t dst, mgfwa_ctx_t src);

/* ---- measurement -------------------------------------------------------- */
/* Times the dominant kernel of a generation in isolation on the context
 * stream with CUDA events: the spark fitness (tcgen05 GEMM for the NN
 * objectives, the fused explode+fitness kernel for analytic ones), `iters`
 * launches after one warm-up, each from a cold L2 (a 256 MB write precedes
 * every timed launch, outside the events).  *ms = mean ms per launch;
 * *units = candidates (rows) per launch. */
int mgfwa_time_fitness(mgfwa_ctx_t ctx, uint64_t iters, double* ms,
                       uint64_t* units);

/* Same, for one kernel of the generation (state-idempotent ones only):
 * MGFWA_KERNEL_FITNESS (as above), _EXPLODE (explode + mapping (+ analytic
 * fitness)), _RANK (spark fitness finalize + ranking), _GUIDES (guiding
 * vector + guides + mapping), _GUIDE_FITNESS (NN fitness of the guides),
 * _SELECT (select_best + update_amplitudes + winner copy; the state it writes
 * is restored before every timed launch and afterwards, so each launch sees
 * the same post-guide pre-selection state).  *units = fireworks for _SELECT.
 * Run on the state the context holds (e.g. after some generations). */
#define MGFWA_KERNEL_FITNESS 0
#define MGFWA_KERNEL_EXPLODE 1
#define MGFWA_KERNEL_RANK 2
#define MGFWA_KERNEL_GUIDES 3
#define MGFWA_KERNEL_GUIDE_FITNESS 4
#define MGFWA_KERNEL_SELECT 5
int mgfwa_time_kernel(mgfwa_ctx_t ctx, int kernel, uint64_t iters, double* ms,
                      uint64_t* units);

/* ---- utilities ---------------------------------------------------------- */
/* MgfwaConfig::validate (config.cpp:42-79): MGFWA_OK, or MGFWA_EINVAL with
 * the reference's message in mgfwa_last_error(NULL).  Host-only, no GPU. */
int mgfwa_validate_config(const mgfwa_config_t* config);
/* key_hash, rng.hpp:43-52, evaluated on the device for n keys [n][7]. */
int mgfwa_key_hash(const uint64_t* keys, uint64_t n, uint64_t* out);
const char* mgfwa_version(void);
/* A destroyed context parks its device workspace (buffers, stream, pinned
 * control block, captured generation graph) for reuse by the next context
 * of the same shape (one entry).  This frees it: the next mgfwa_create /
 * mgfwa_run_once then pays the full setup (allocation, dataset, TMA
 * descriptors, graph capture). */
int mgfwa_release_cached_workspace(void);

#ifdef __cplusplus
}
#endif

#endif /* MGFWA_B200_H */
