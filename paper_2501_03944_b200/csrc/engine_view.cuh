// engine_view.cuh — the device-side view of one engine context.
//
// HBM layout (all row-major, rows padded to Dp = round_up(D, 64) elements so
// every row starts 256-byte aligned and bf16 rows are TMA-addressable):
//   pos      float [F][Dp]        firework positions (F = B * mu)
//   sparks   float [F*lam][Dp]    explosion sparks, row n*lam+k per batch
//   sparks_h bf16  [F*lam][Dp]    bf16 shadow (NN objectives only)
//   guides   float [F*M][Dp]      guiding sparks, row n*M+m per batch
//   fresh_h  bf16  [F][Dp]        reinit / init rows for NN evaluation
//   *part    float [rows][nparts][2]  per-chunk fitness partial sums
// Scalars per firework (fit, amp, li) are fp64: they are tiny and keep the
// selection / amplitude / loser-out arithmetic identical to the reference.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace mgfwa_b200 {

constexpr uint64_t kMaxSparksPerFirework = 16384;  // k_rank keys in shared memory
constexpr int kChunk = 512;  // coordinates per warp work item (32 lanes x 4 x 4)

struct Ctl {
  uint64_t iteration;     // iteration of the generation about to run (1-based)
  uint64_t used;          // evaluations_used
  uint64_t losers_total;  // losers_reinitialized
  uint64_t nan_count;     // nan_evaluations
  uint64_t trace_n;       // trace waves written so far
  uint64_t start_ns;      // %globaltimer at the start of initialize()
  uint64_t gens_run;      // loop bodies executed
  double init_ms;         // elapsed at the end of initialize()
  double iters_rem;       // iterations_remaining of the current generation
  int active;             // 1 while the loop body must run
  int n_losers;           // losers of the current generation
  unsigned small_done;    // blocks of k_small_b done in this generation
  unsigned bar_count;     // grid barrier of the persistent small-problem loop
  unsigned bar_gen;
  uint64_t n_losers_all;  // replica sharding: losers of the generation over all shards
  // sharded runs (EngineView::nan_mode != 0): NaN evaluations of work only
  // this shard did (phase A; replica mode: also its own losers) go to
  // nan_own; the exchange brings the other shards' counts into nan_all
  // (NCCL: the all-reduced total), and k_finalize_record(1) folds them into
  // nan_count, so nan_evaluations is the global count on every shard.
  uint64_t nan_own;
  uint64_t nan_all;
};

struct EngineView {
  // shape.  F = B * mu fireworks in total; this context owns the contiguous
  // range [f_lo, f_lo + Fl) (firework sharding across ranks).
  // Spark / guide buffers hold only the owned fireworks (local row
  // (f - f_lo) * lam + k); positions, fitness, amplitudes and improvement
  // rates are replicated for all F (refreshed by the per-generation
  // all-gather), so population range, loser-out and record_wave run
  // identically on every rank.
  uint64_t B, mu, lam, M, D, Dp, top, F;
  uint64_t Fl, f_lo;
  // replica sharding (MGFWA_SHARD_REPLICA): the owned fireworks are whole
  // batches [b_lo, b_hi); loser-out, record_wave and the population range run
  // for those batches only and the shards exchange just the loser count.
  int replica;
  uint64_t b_lo, b_hi;
  // NaN accounting across shards: 0 unsharded, 1 emulated shards (in-process
  // exchange adds the peers' nan_own), 2 NCCL (all-reduced nan_own).
  int nan_mode;
  uint32_t nparts;     // partial-sum slots per row
  uint32_t nch;        // coordinate chunks per row (kChunk each)
  int obj_kind;
  int nn;              // 1 when fitness runs on the tensor cores
  uint32_t samples;    // NN: S
  uint64_t seed;
  // algorithm parameters (MgfwaConfig)
  double amp_amplify, amp_reduce, a0, max_range, amp_floor;
  uint64_t max_evals;
  double wall_budget_ms;
  uint64_t wave;
  // search space
  const double* lower;
  const double* upper;
  const float* lower_f;  // smallest float >= lower[d]
  const float* upper_f;  // largest  float <= upper[d]
  const double* boosts;  // [M]
  // state
  float* pos;
  double* fit;
  double* fit_prev;  // pre-selection firework fitness (k_rank), read by every k_select part
  double* amp;
  double* li;
  int* improved;
  int* winner;
  int* loser;
  float* pop_lo;  // [B][Dp]
  float* pop_hi;
  float* sparks;
  __nv_bfloat16* sparks_h;
  float* sfit;
  float* spart;
  int* rank_idx;  // [F][2*top]: top (best first) then bottom (rank order)
  float* guides;
  __nv_bfloat16* guides_h;
  float* gfit;
  float* gpart;
  __nv_bfloat16* fresh_h;
  float* fpart;
  double* best_fit;  // [B]
  float* best_pos;   // [B][Dp]
  int* best_idx;     // [B]
  int* rec_flag;     // [B]
  uint64_t* tr_evals;  // [cap][B]
  double* tr_best;
  uint64_t* tr_ns;
  uint64_t trace_cap;
  Ctl* ctl;
  // operator-seam switches (tests): fitness given by the caller instead of
  // the partial sums, and a fixed iterations_remaining for loser_out.
  int injected_fitness;
  int has_iters_override;
  double iters_override;
  // test switch (MGFWA_EXPLODE_GENERAL=1): every explode draw through the
  // general key form (mix_draw), never the chunk-constant one (chunk_draw),
  // so the parity tests reach the path a near-carry chunk takes
  int explode_general;
};

}  // namespace mgfwa_b200
