// kernels.h — host-side launch entry points of the device kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "engine_view.cuh"

namespace mgfwa_b200 {

// Tensor-core fitness calls the engine interleaves with its own kernels.
struct GenerationHooks {
  void* ctx;
  void (*eval_sparks)(void* ctx, cudaStream_t s);
  void (*eval_guides)(void* ctx, cudaStream_t s);
  void (*eval_fresh)(void* ctx, cudaStream_t s);      // gated on n_losers
  void (*eval_fresh_all)(void* ctx, cudaStream_t s);  // initialize()
  // optional: explode + spark fitness as one pipelined step (replaces the
  // explode launch and eval_sparks; see launch_explode_fireworks)
  void (*explode_eval)(void* ctx, cudaStream_t s);
};

// One-time kernel attributes (dynamic shared memory opt-in); call before
// the first launch / graph capture.
cudaError_t prepare_engine_kernels();

enum { kGenAll = 0, kGenA = 1, kGenB = 2 };
void launch_generation_kernels(const EngineView& v, int nsm, cudaStream_t s,
                               GenerationHooks* hooks, int phase = kGenAll);
void launch_initialize_kernels(const EngineView& v, int nsm, cudaStream_t s,
                               GenerationHooks* hooks);

// Persistent whole-loop kernel for small analytic problems (one context,
// D <= 512, B * mu <= #SMs): up to max_gens generations in one cooperative launch.
bool small_run_ok(const EngineView& v, int nsm);
cudaError_t launch_small_run(const EngineView& v, uint64_t max_gens, cudaStream_t s);

// operator seams
void launch_pop_range(const EngineView& v, int nsm, cudaStream_t s);
void launch_explode_map(const EngineView& v, int nsm, cudaStream_t s);
void launch_explode_fireworks(const EngineView& v, uint64_t f0, uint64_t nf, int nsm, cudaStream_t s);
void launch_rank(const EngineView& v, cudaStream_t s);
void launch_guides(const EngineView& v, int nsm, cudaStream_t s);
void launch_select(const EngineView& v, int nsm, cudaStream_t s);
void launch_select_gen(const EngineView& v, int nsm, cudaStream_t s);
void launch_loser(const EngineView& v, int nsm, cudaStream_t s);
void launch_loser_commit(const EngineView& v, int nsm, cudaStream_t s);
void launch_analytic_partials(const float* rows, uint64_t nrows, uint64_t D,
                              uint64_t Dp, uint32_t nch, int kind, float* part,
                              int nsm, cudaStream_t s);
void launch_finalize_rows(const EngineView& v, const float* part,
                          uint64_t nrows, float* fitness,
                          unsigned long long* nan, cudaStream_t s);
void launch_map_rows(const EngineView& v, const float* cand, float* out,
                     uint64_t rows, uint64_t per, uint64_t stream, uint64_t it,
                     cudaStream_t s);
void launch_argmin_rows(const double* fit, uint64_t rows, uint64_t cols,
                        uint64_t* idx, double* val, cudaStream_t s);
void launch_key_hash(const uint64_t* keys, uint64_t n, uint64_t* out,
                     cudaStream_t s);
// dst->n_losers_all += src->n_losers (when losers), dst->nan_all += src->nan_own
void launch_add_losers(Ctl* dst, const Ctl* src, int losers, cudaStream_t s);
// ctl->nan_count += ctl->nan_all; nan_own = nan_all = 0 (after an all-reduce of nan_own)
void launch_fold_nan(Ctl* ctl, cudaStream_t s);
void launch_to_bf16(const float* src, __nv_bfloat16* dst, uint64_t n,
                    cudaStream_t s);

// ---- tensor-core MLP fitness (k_mlp_tc.cu) ----
// Opaque plan: TMA descriptors for the shared dataset X [S][I] and for one
// candidate buffer W (bf16 rows of stride Dp holding W1 [H][I] at offset 0,
// then b1, W2 [O][H], b2).
struct MlpPlan;
// Returns nullptr and fills err on an unsupported shape.
MlpPlan* mlp_plan_create(const __nv_bfloat16* X, const int32_t* y,
                         uint32_t S, uint32_t I, uint32_t H, uint32_t O,
                         const __nv_bfloat16* W, uint64_t rows, uint64_t Dp,
                         int nsm, char* err, size_t errlen);
void mlp_plan_destroy(MlpPlan* p);
// part[row][m_tile][2] (slot 0 = sum of CE over the m-tile's samples).
// gate: if non-null and *gate == 0 the kernel exits immediately.
// launch_done (optional): recorded once every CTA of the launch is resident
// (cudaLaunchAttributeLaunchCompletionEvent)
cudaError_t mlp_fitness_launch(const MlpPlan* p, float* part,
                               const int* gate, cudaStream_t s, cudaEvent_t launch_done = nullptr);
uint32_t mlp_num_parts(uint32_t S);

// ---- LeNet-5 fitness (k_lenet.cu, warp-level bf16 MMA) ----
// W rows of stride Dp hold the 61,706 LeNet parameters (oracle f_lenet
// order); X [S][784] bf16, y [S].  part[row][chunk of 128 samples][2].
struct LenetPlan;
LenetPlan* lenet_plan_create(const __nv_bfloat16* X, const int32_t* y, uint32_t S,
                             const __nv_bfloat16* W, uint64_t rows, uint64_t Dp, int nsm,
                             char* err, size_t errlen);
void lenet_plan_destroy(LenetPlan* p);
cudaError_t lenet_fitness_launch(const LenetPlan* p, float* part, const int* gate,
                                 cudaStream_t s);
uint32_t lenet_num_parts(uint32_t S);
uint64_t lenet_dim();

// ---- reference benchmark networks (k_net.cu, fp64 layer GEMMs) ----
// X: fp32 candidate rows of stride ldx; part[row][1][2] = network output.
struct NetPlan;
bool net_spec_dims(int net_id, uint32_t* input_dim, uint32_t* hidden_dim, uint32_t* layers,
                   int* gelu);
NetPlan* net_plan_create(int net_id, uint64_t weight_seed, const float* X, uint64_t ldx,
                         uint64_t rows, char* err, size_t errlen);
void net_plan_destroy(NetPlan* p);
cudaError_t net_fitness_launch(const NetPlan* p, float* part, const int* gate, cudaStream_t s);

}  // namespace mgfwa_b200
