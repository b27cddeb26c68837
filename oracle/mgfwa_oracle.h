/*
 * mgfwa_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, fp64 restatement of the reference MGFWA generation path
 * (/root/reference/proj, C++20, CPU-only).  It is the checker the parity
 * tests, __graft_entry__.smoke() and bench.py's cpu_baseline leg compare the
 * B200 engine against.  It is never linked into, loaded by, or called from
 * the product library (paper_2501_03944_b200/libmgfwa_b200.so).
 *
 * Pinned by: tests/golden/*.json, generated from the compiled reference
 * (oracle/_ref/libmgfwa_ref.so built by oracle/Makefile from the reference
 * sources) by tests/golden/make_golden.py, and checked in
 * tests/test_oracle_golden.py.  The restated objectives that the reference
 * does not ship (Rastrigin, Ackley, MLP-weights loss, LeNet loss) are
 * "parity unpinned" against the reference itself; they are pinned by
 * known-answer values and by agreement with a second independent C++
 * restatement inside oracle/ref_shim.cpp.
 */
#ifndef MGFWA_ORACLE_H
#define MGFWA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* RngStream, rng.hpp:11-18 (+ kData = 7, builder-defined synthetic data). */
enum {
  ORC_INIT = 1,
  ORC_EXPLODE = 2,
  ORC_MAPPING = 3,
  ORC_GUIDE = 4,
  ORC_REINIT = 5,
  ORC_WEIGHTS = 6,
  ORC_DATA = 7
};

/* Objective kinds (mirror include/mgfwa_b200.h). */
enum {
  ORC_OBJ_SPHERE = 1,
  ORC_OBJ_RASTRIGIN = 2,
  ORC_OBJ_ACKLEY = 3,
  ORC_OBJ_MLP_WEIGHTS = 4,
  ORC_OBJ_LENET = 5,
  ORC_OBJ_NET = 6 /* reference input-space MlpBlackBox (nets.cpp:138-167) */
};

/* MgfwaConfig, config.hpp:33-47. */
typedef struct {
  uint64_t batches;
  uint64_t fireworks;
  uint64_t sparks;
  uint64_t guides;
  double guide_fraction;
  const double* boosts; /* length == guides */
  uint64_t n_boosts;
  double amp_amplify;
  double amp_reduce;
  double initial_amplitude;
  uint64_t max_evaluations;
  double wall_clock_budget_ms;
} orc_config_t;

typedef struct orc_objective orc_objective_t;

/* ---- rng.hpp:33-65 ---- */
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_key_hash(uint64_t seed, uint64_t stream, uint64_t iteration,
                      uint64_t b, uint64_t n, uint64_t k, uint64_t d);
double orc_unit_uniform(uint64_t seed, uint64_t stream, uint64_t iteration,
                        uint64_t b, uint64_t n, uint64_t k, uint64_t d);
/* returns 0, or -1 when !(lo <= hi) (rng.hpp:61-63) */
int orc_uniform_sample(uint64_t seed, uint64_t stream, uint64_t iteration,
                       uint64_t b, uint64_t n, uint64_t k, uint64_t d,
                       double lo, double hi, double* out);

/* ---- config.cpp ---- */
uint64_t orc_top_spark_count(const orc_config_t* c);
/* NULL when valid, else the reference's exception message. */
const char* orc_config_validate(const orc_config_t* c);
const char* orc_space_validate(const double* lower, const double* upper,
                               uint64_t dim);
double orc_max_range(const double* lower, const double* upper, uint64_t dim);

/* ---- objectives ---- */
orc_objective_t* orc_objective_create(int kind, uint32_t in_dim,
                                      uint32_t hidden, uint32_t out_dim,
                                      uint32_t samples, uint64_t data_seed);
void orc_objective_destroy(orc_objective_t* obj);
uint64_t orc_objective_dim(const orc_objective_t* obj);
double orc_objective_eval(const orc_objective_t* obj, const double* x,
                          uint64_t dim);
/* synthetic dataset (kData stream): X[S*784-like in_dim], y[S] */
void orc_make_dataset(uint32_t samples, uint32_t in_dim, uint32_t out_dim,
                      uint64_t data_seed, double* X, int32_t* y);
const double* orc_objective_data(const orc_objective_t* obj);
const int32_t* orc_objective_labels(const orc_objective_t* obj);

/* batched_apply, backend.cpp:28-67: NaN -> +inf, returns #NaN. */
uint64_t orc_batched_apply(const orc_objective_t* obj, const double* rows,
                           uint64_t nrows, uint64_t dim, double* fitness);
/* argmin_per_population, backend.cpp:69-83 */
void orc_argmin_per_population(const double* fitness, uint64_t rows,
                               uint64_t cols, uint64_t* index, double* value);

/* ---- engine.cpp operators ---- */
void orc_population_range(const double* pos, uint64_t B, uint64_t mu,
                          uint64_t D, double* lo, double* hi);
void orc_initialize_positions(const orc_config_t* c, const double* lower,
                              const double* upper, uint64_t D, uint64_t seed,
                              double* pos);
void orc_explode(const double* pos, const double* amp, uint64_t B,
                 uint64_t mu, uint64_t D, uint64_t lambda, uint64_t iteration,
                 uint64_t seed, double* sparks);
void orc_random_mapping(double* cand, uint64_t B, uint64_t rows, uint64_t D,
                        uint64_t per, const double* pos, uint64_t mu,
                        const double* lower, const double* upper,
                        uint64_t iteration, uint64_t seed, uint64_t stream);
/* returns 0 or -1 (lambda < 2*top) */
int orc_guiding_vector(const double* sparks, const double* spark_fit,
                       uint64_t B, uint64_t mu, uint64_t lambda, uint64_t D,
                       uint64_t top, double* delta);
void orc_multi_guiding_sparks(const double* pos, const double* delta,
                              uint64_t B, uint64_t mu, uint64_t D,
                              const double* boosts, uint64_t M,
                              double* guides);
/* guides may be NULL (M = 0). Writes new pos/fit/li and improved. */
void orc_select_best(const double* pos, const double* fit, uint64_t B,
                     uint64_t mu, uint64_t D, const double* sparks,
                     const double* spark_fit, uint64_t lambda,
                     const double* guides, const double* guide_fit,
                     uint64_t M, double* new_pos, double* new_fit,
                     double* new_li, double* improved);
void orc_update_amplitudes(const double* amp, const double* improved,
                           uint64_t n, double amp_amplify, double amp_reduce,
                           double max_range, double* out);
/* In-place on pos/fit/amp/li; returns #losers; *nan_count += NaNs. */
uint64_t orc_loser_out(double* pos, double* fit, double* amp, double* li,
                       uint64_t B, uint64_t mu, uint64_t D,
                       const orc_config_t* c, const double* lower,
                       const double* upper, uint64_t iteration, uint64_t seed,
                       double iterations_remaining, const orc_objective_t* obj,
                       uint64_t* nan_count);

typedef struct {
  uint64_t evaluations_used;
  uint64_t iterations;
  uint64_t losers_reinitialized;
  uint64_t nan_evaluations;
  uint64_t waves; /* trace points per batch */
} orc_counters_t;

/* run(), engine.cpp:313-423 (max_evaluations budget; the wall-clock budget
 * is honoured with CLOCK_MONOTONIC).  trace arrays are [B][trace_cap].
 * Returns NULL on success or an error message. */
const char* orc_run(const orc_config_t* c, const double* lower,
                    const double* upper, uint64_t D,
                    const orc_objective_t* obj, uint64_t seed,
                    double* best_fitness, double* best_position,
                    uint64_t* trace_evals, double* trace_best,
                    double* trace_wall_ms, uint64_t trace_cap,
                    orc_counters_t* counters);

#ifdef __cplusplus
}
#endif

#endif /* MGFWA_ORACLE_H */
