// engine.cu — host side of the B200 MGFWA engine and its C-ABI
// (include/mgfwa_b200.h).
//
// The Engine owns every device buffer of one run (layout: engine_view.cuh),
// captures one generation (engine.cpp:359-417) as a CUDA graph, and replays
// it; loop control (iteration counter, evaluation accounting, termination)
// lives in a device control block so the host only syncs once per chunk of
// generations.  The reference's run() (engine.cpp:313-423) maps to
// mgfwa_run(); its operators (engine.hpp:71-125) map to mgfwa_op_*.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only; the library is bound at run time (dlopen)

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <functional>
#include <vector>

#include "../../include/mgfwa_b200.h"
#include "common.cuh"
#include "engine_view.cuh"
#include "kernels.h"

namespace mgfwa_b200 {

// ----------------------------------------------------------------- errors
struct Status {
  int code;
  std::string msg;
};

static thread_local std::string g_last_error;

#define CUDA_TRY(expr)                                                        \
  do {                                                                        \
    cudaError_t e__ = (expr);                                                 \
    if (e__ != cudaSuccess)                                                   \
      return Status{MGFWA_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)}; \
  } while (0)

#define STATUS_TRY(expr)                      \
  do {                                        \
    Status s__ = (expr);                      \
    if (s__.code != MGFWA_OK) return s__;     \
  } while (0)

static Status ok() { return Status{MGFWA_OK, ""}; }
static Status invalid(const std::string& m) { return Status{MGFWA_EINVAL, m}; }

// --------------------------------------------------------- config checks
struct HostConfig {
  uint64_t B = 8, mu = 5, lam = 30, M = 3;
  double sigma = 0.2;
  std::vector<double> boosts{1.0, 2.0, 4.0};
  double amp_amplify = 1.2, amp_reduce = 0.9, a0 = 0.0;
  uint64_t max_evals = 0;
  double wall_ms = 0.0;
  uint64_t top() const { return (uint64_t)std::ceil(sigma * (double)lam); }
  uint64_t wave() const { return B * mu * (lam + M); }
};

static HostConfig to_host(const mgfwa_config_t* c) {
  HostConfig h;
  h.B = c->batches;
  h.mu = c->fireworks;
  h.lam = c->sparks_per_firework;
  h.M = c->guides_per_firework;
  h.sigma = c->guide_fraction;
  h.boosts.assign(c->boosts, c->boosts + (c->boosts ? c->n_boosts : 0));
  h.amp_amplify = c->amp_amplify;
  h.amp_reduce = c->amp_reduce;
  h.a0 = c->initial_amplitude;
  h.max_evals = c->max_evaluations;
  h.wall_ms = c->wall_clock_budget_ms;
  return h;
}

// MgfwaConfig::validate, config.cpp:42-79 (same messages, same order).
static Status validate_config(const HostConfig& c) {
  if (c.B == 0 || c.mu == 0 || c.lam == 0)
    return invalid("MgfwaConfig: batches, fireworks and sparks must be positive");
  if (!(c.amp_amplify > 1.0)) return invalid("MgfwaConfig: amp_amplify must be > 1");
  if (!(c.amp_reduce > 0.0 && c.amp_reduce < 1.0))
    return invalid("MgfwaConfig: amp_reduce must be in (0, 1)");
  if (c.max_evals == 0 && !(c.wall_ms > 0.0))
    return invalid("MgfwaConfig: at least one budget must be positive");
  if (c.M > 0) {
    if (!(c.sigma > 0.0 && c.sigma <= 0.5))
      return invalid("MgfwaConfig: guide_fraction must be in (0, 0.5]");
    if (c.sigma * (double)c.lam < 1.0)
      return invalid("MgfwaConfig: guide_fraction * sparks must be >= 1");
    if (c.lam < 2 * c.top())
      return invalid(
          "MgfwaConfig: sparks must cover disjoint elite and poor sets "
          "(lambda >= 2 * ceil(sigma * lambda))");
    if (c.boosts.size() != c.M)
      return invalid("MgfwaConfig: boosts must list one coefficient per guide");
    if (c.boosts.front() != 1.0) return invalid("MgfwaConfig: first boost coefficient must be 1");
    for (double b : c.boosts)
      if (!(b > 0.0) || !std::isfinite(b))
        return invalid("MgfwaConfig: boost coefficients must be positive finite");
    if (c.M > 16) return invalid("mgfwa_b200: guides_per_firework > 16 is not supported");
  }
  // k_rank keeps one 8-byte key per spark in shared memory on every
  // generation, with or without guides
  if (c.lam > kMaxSparksPerFirework)
    return invalid("mgfwa_b200: sparks_per_firework > 16384 is not supported");
  return ok();
}

// SearchSpace::validate, config.cpp:25-35.
static Status validate_space(const mgfwa_space_t* s) {
  if (s == nullptr || s->dim == 0 || s->lower == nullptr || s->upper == nullptr)
    return invalid("SearchSpace: lower/upper must be non-empty and equal length");
  for (uint64_t d = 0; d < s->dim; ++d)
    if (!std::isfinite(s->lower[d]) || !std::isfinite(s->upper[d]) || !(s->lower[d] < s->upper[d]))
      return invalid("SearchSpace: requires lower[d] < upper[d] for all d");
  return ok();
}

// NN objectives (tensor-core fitness): the MLP-weights loss and LeNet-5.
// NN fitness path (partials from a fitness kernel, not fused into explode):
// the MLP-weights and LeNet losses (synthetic dataset) and the reference's
// input-space benchmark networks (fixed weights).
static bool nn_kind(int kind) {
  return kind == MGFWA_OBJ_MLP_WEIGHTS || kind == MGFWA_OBJ_LENET || kind == MGFWA_OBJ_NET;
}
static bool has_dataset(int kind) { return kind == MGFWA_OBJ_MLP_WEIGHTS || kind == MGFWA_OBJ_LENET; }
static uint32_t nn_in_dim(const mgfwa_objective_t* o) {
  return o->kind == MGFWA_OBJ_LENET ? 784u : o->in_dim;
}
static uint32_t nn_out_dim(const mgfwa_objective_t* o) {
  return o->kind == MGFWA_OBJ_LENET ? 10u : o->out_dim;
}

// One NN fitness plan: the MLP (tcgen05), LeNet (mma.sync) or benchmark
// network (fp64 GEMM chain) kernel.
struct NnPlan {
  MlpPlan* mlp = nullptr;
  LenetPlan* lenet = nullptr;
  NetPlan* net = nullptr;
  void destroy() {
    mlp_plan_destroy(mlp);
    lenet_plan_destroy(lenet);
    net_plan_destroy(net);
    mlp = nullptr;
    lenet = nullptr;
    net = nullptr;
  }
};
static cudaError_t nn_fitness_launch(const NnPlan& p, float* part, const int* gate,
                                     cudaStream_t s) {
  if (p.net) return net_fitness_launch(p.net, part, gate, s);
  return p.lenet ? lenet_fitness_launch(p.lenet, part, gate, s)
                 : mlp_fitness_launch(p.mlp, part, gate, s);
}

static uint64_t objective_dim(const mgfwa_objective_t* o) {
  if (o->kind == MGFWA_OBJ_LENET) return lenet_dim();
  if (o->kind == MGFWA_OBJ_NET) {
    uint32_t d = 0;
    net_spec_dims(o->net_id, &d, nullptr, nullptr, nullptr);
    return d;
  }
  if (o->kind == MGFWA_OBJ_MLP_WEIGHTS)
    return (uint64_t)o->hidden * o->in_dim + o->hidden + (uint64_t)o->out_dim * o->hidden +
           o->out_dim;
  return 0;
}

static Status validate_objective(const mgfwa_objective_t* o, uint64_t D) {
  if (o == nullptr) return invalid("batched_apply: empty objective");
  switch (o->kind) {
    case MGFWA_OBJ_SPHERE:
    case MGFWA_OBJ_RASTRIGIN:
    case MGFWA_OBJ_ACKLEY:
      return ok();
    case MGFWA_OBJ_MLP_WEIGHTS:
      if (o->samples == 0 || o->in_dim == 0 || o->hidden == 0 || o->out_dim == 0)
        return invalid("MLP objective: all dimensions must be positive");
      if (objective_dim(o) != D)
        return invalid("forward: input dimension mismatch");
      return ok();
    case MGFWA_OBJ_LENET:
      if (o->samples == 0) return invalid("LeNet objective: samples must be positive");
      if (objective_dim(o) != D) return invalid("forward: input dimension mismatch");
      return ok();
    case MGFWA_OBJ_NET:  // net_spec (nets.cpp:57-62), forward (nets.cpp:138-141)
      if (o->net_id < 1 || o->net_id > 12) return invalid("net id must be in 1..12");
      if (objective_dim(o) != D) return invalid("forward: input dimension mismatch");
      return ok();
    default:
      return invalid("unknown objective kind");
  }
}

// Builder-defined synthetic dataset (kData stream; oracle/mgfwa_oracle.c
// orc_make_dataset restates the same definition): 8-bit pixels
// X = (H(seed,kData,0,0,s,0,i) >> 56) / 256 (exact in bf16), labels from a
// random linear teacher, fp64 host arithmetic in the same order.
static void make_dataset(uint32_t S, uint32_t I, uint32_t O, uint64_t seed,
                         std::vector<__nv_bfloat16>& Xh, std::vector<int32_t>& y) {
  std::vector<double> T((size_t)O * I), X((size_t)S * I);
  for (uint32_t o = 0; o < O; ++o)
    for (uint32_t i = 0; i < I; ++i) {
      const uint64_t h = splitmix64(key_prefix(seed, kData, 1, 0, o, 0) ^ i);
      const double u = (double)(h >> 11) * 0x1.0p-53;
      T[(size_t)o * I + i] = -1.0 + u * (1.0 - -1.0);
    }
  Xh.resize((size_t)S * I);
  y.resize(S);
  for (uint32_t s = 0; s < S; ++s) {
    const uint64_t pre = key_prefix(seed, kData, 0, 0, s, 0);
    for (uint32_t i = 0; i < I; ++i) {
      const double x = (double)(splitmix64(pre ^ i) >> 56) / 256.0;
      X[(size_t)s * I + i] = x;
      Xh[(size_t)s * I + i] = __float2bfloat16_rn((float)x);
    }
    int32_t best = 0;
    double best_v = 0.0;
    for (uint32_t o = 0; o < O; ++o) {
      double acc = 0.0;
      for (uint32_t i = 0; i < I; ++i) acc += T[(size_t)o * I + i] * (X[(size_t)s * I + i] - 0.5);
      if (o == 0 || acc > best_v) best_v = acc, best = (int32_t)o;
    }
    y[s] = best;
  }
}

static float f32_ceil_of(double x) {  // smallest float >= x
  float f = (float)x;
  if ((double)f < x) f = std::nextafter(f, std::numeric_limits<float>::infinity());
  return f;
}
static float f32_floor_of(double x) {  // largest float <= x
  float f = (float)x;
  if ((double)f > x) f = std::nextafter(f, -std::numeric_limits<float>::infinity());
  return f;
}

static uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// ------------------------------------------------------------- workspace
// One device arena holding every buffer of a run; builds the EngineView.
struct Workspace {
  EngineView v{};
  void* arena = nullptr;
  size_t arena_bytes = 0;
  __nv_bfloat16* X = nullptr;  // NN dataset
  int32_t* y = nullptr;
  NnPlan plan_sparks, plan_guides, plan_fresh;
  // pipelined explode -> spark fitness (MLP objective): fitness plans over
  // firework chunks [chunk_f0[c], + chunk_nf[c]) of the owned fireworks, an
  // auxiliary stream the explode chunks run on, and fork/join events
  std::vector<NnPlan> plan_chunks;
  std::vector<uint64_t> chunk_f0, chunk_nf;
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr;
  std::vector<cudaEvent_t> ev_chunk, ev_launched;
  bool pipe_lc = false;  // explode chunk c+1 waits for the launch (not the end) of fitness chunk c
  int nsm = 148;
  int device = 0;

  // per-workspace host/stream resources and the last captured generation
  // graph (reused by the next run on this workspace when its EngineView —
  // every by-value kernel argument — is unchanged)
  cudaStream_t stream = nullptr;
  Ctl* host_ctl = nullptr;  // pinned
  cudaGraphExec_t exec_all = nullptr;
  std::vector<unsigned char> exec_view;
  size_t exec_nodes = 0;

  ~Workspace() {
    if (exec_all) cudaGraphExecDestroy(exec_all);
    if (stream) cudaStreamDestroy(stream);
    if (host_ctl) cudaFreeHost(host_ctl);
    plan_sparks.destroy();
    plan_guides.destroy();
    plan_fresh.destroy();
    for (auto& pc : plan_chunks) pc.destroy();
    for (auto e : ev_chunk) cudaEventDestroy(e);
    for (auto e : ev_launched) cudaEventDestroy(e);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (aux) cudaStreamDestroy(aux);
    if (arena) cudaFree(arena);
  }

  // Pipelined explode -> fitness (MLP-weights objective): up to 8 chunks of
  // whole fireworks, used when every chunk holds >= 4096 sparks (C5: 8 x
  // 8 x 1024; 82.5 -> 78.4 ms per generation).  Small populations lose more
  // to the extra fitness launches than the overlap gains (C2: 309 -> 366
  // us), so they keep one explode and one fitness launch.  MGFWA_PIPELINE=0
  // / =1 force it off / on.
  Status build_pipeline(const mgfwa_objective_t* obj) {
    const char* env = getenv("MGFWA_PIPELINE");
    if (obj->kind != MGFWA_OBJ_MLP_WEIGHTS || v.Fl < 2) return ok();
    const uint64_t G = std::min<uint64_t>(v.Fl, 8);
    const bool large = (v.Fl / G) * v.lam >= 4096;
    if (env ? env[0] == '0' : !large) return ok();
    char err[256] = {0};
    for (uint64_t c = 0; c < G; ++c) {
      const uint64_t f0 = v.Fl * c / G, f1 = v.Fl * (c + 1) / G;
      NnPlan pl;
      pl.mlp = mlp_plan_create(X, y, obj->samples, obj->in_dim, obj->hidden, obj->out_dim,
                               v.sparks_h + f0 * v.lam * v.Dp, (f1 - f0) * v.lam, v.Dp, nsm, err, sizeof err);
      if (!pl.mlp) return invalid(err);
      plan_chunks.push_back(pl);
      chunk_f0.push_back(f0);
      chunk_nf.push_back(f1 - f0);
      cudaEvent_t e, l;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&l, cudaEventDisableTiming));
      ev_chunk.push_back(e);
      ev_launched.push_back(l);
    }
    // launch-completion edges (explode c+1 released when fitness c is resident)
    // measured slower (C2 407 vs 366 us, C5 80.2 vs 78.4 ms): off unless =1
    const char* lc = getenv("MGFWA_PIPELINE_LC");
    pipe_lc = lc && lc[0] == '1';
    CUDA_TRY(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    CUDA_TRY(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
    return ok();
  }

  // Everything that sizes device memory or the dataset; workspaces with an
  // equal key are reused across runs (see WorkspaceCache).
  std::vector<uint64_t> key;

  static std::vector<uint64_t> make_key(const HostConfig& c, const mgfwa_space_t* space,
                                        const mgfwa_objective_t* obj, int dev, uint64_t trace_cap,
                                        uint64_t rank = 0, uint64_t world = 1) {
    return {c.B, c.mu, c.lam, c.M, c.M > 0 ? c.top() : 0, space->dim, (uint64_t)obj->kind,
            obj->in_dim, obj->hidden, obj->out_dim, obj->samples,
            nn_kind(obj->kind) ? obj->data_seed : 0, (uint64_t)dev, trace_cap,
            rank, world, obj->kind == MGFWA_OBJ_NET ? (uint64_t)obj->net_id : 0,
            obj->kind == MGFWA_OBJ_NET ? obj->weight_seed : 0};
  }

  // Run-specific scalars and the search box (cheap; H2D of 2 x D bounds).
  Status configure(const HostConfig& c, const mgfwa_space_t* space, uint64_t seed) {
    const uint64_t D = space->dim;
    v.seed = seed;
    v.replica = 0;  // firework sharding (the default); mgfwa_set_shard_mode switches
    v.b_lo = 0;
    v.b_hi = c.B;
    v.amp_amplify = c.amp_amplify;
    v.amp_reduce = c.amp_reduce;
    double max_range = 0.0;
    for (uint64_t d = 0; d < D; ++d) max_range = std::max(max_range, space->upper[d] - space->lower[d]);
    v.max_range = max_range;
    v.amp_floor = 1e-12 * max_range;
    v.a0 = c.a0 > 0.0 ? c.a0 : 0.5 * max_range;
    v.max_evals = c.max_evals;
    v.wall_budget_ms = c.wall_ms;
    v.wave = c.wave();
    v.injected_fitness = 0;
    v.has_iters_override = 0;
    std::vector<float> lf(D), uf(D);
    for (uint64_t d = 0; d < D; ++d) {
      lf[d] = f32_ceil_of(space->lower[d]);
      uf[d] = f32_floor_of(space->upper[d]);
    }
    CUDA_TRY(cudaSetDevice(device));
    CUDA_TRY(cudaMemcpy(const_cast<double*>(v.lower), space->lower, D * 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(const_cast<double*>(v.upper), space->upper, D * 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(const_cast<float*>(v.lower_f), lf.data(), D * 4, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(const_cast<float*>(v.upper_f), uf.data(), D * 4, cudaMemcpyHostToDevice));
    if (v.M > 0)
      CUDA_TRY(cudaMemcpy(const_cast<double*>(v.boosts), c.boosts.data(), v.M * 8, cudaMemcpyHostToDevice));
    return ok();
  }

  Status build(const HostConfig& c, const mgfwa_space_t* space, const mgfwa_objective_t* obj,
               uint64_t seed, int dev, uint64_t trace_cap, uint64_t rank = 0,
               uint64_t world = 1) {
    device = dev;
    key = make_key(c, space, obj, dev, trace_cap, rank, world);
    CUDA_TRY(cudaSetDevice(dev));
    CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CUDA_TRY(prepare_engine_kernels());
    const uint64_t D = space->dim;
    v.B = c.B;
    v.mu = c.mu;
    v.lam = c.lam;
    v.M = c.M;
    v.D = D;
    v.Dp = round_up(D, 64);
    v.top = c.M > 0 ? c.top() : 0;
    {
      const char* eg = getenv("MGFWA_EXPLODE_GENERAL");  // test switch, engine_view.cuh
      v.explode_general = eg != nullptr && eg[0] == '1';
    }
    v.F = c.B * c.mu;
    if (world == 0 || v.F % world != 0)
      return invalid("mgfwa_b200: batches * fireworks must be divisible by the number of ranks");
    v.Fl = v.F / world;
    v.f_lo = rank * v.Fl;
    v.nch = (uint32_t)((D + kChunk - 1) / kChunk);
    v.obj_kind = obj->kind;
    v.nn = nn_kind(obj->kind);
    v.samples = !v.nn ? 0 : obj->kind == MGFWA_OBJ_NET ? 1 : obj->samples;
    v.nparts = !v.nn                         ? v.nch
               : obj->kind == MGFWA_OBJ_NET   ? 1
               : obj->kind == MGFWA_OBJ_LENET ? lenet_num_parts(obj->samples)
                                              : mlp_num_parts(obj->samples);
    v.trace_cap = trace_cap;

    // ---- arena layout
    struct Slot {
      void** dst;
      size_t bytes;
    };
    std::vector<Slot> slots;
    auto add = [&](auto** p, size_t bytes) { slots.push_back({reinterpret_cast<void**>(p), bytes}); };
    // sparks / guides / rank lists for the owned fireworks only
    const uint64_t F = v.F, Dp = v.Dp, P = v.Fl * v.lam, G = v.Fl * v.M, np2 = (uint64_t)v.nparts * 2;
    double *lower, *upper, *boosts;
    float *lower_f, *upper_f;
    add(&lower, D * 8);
    add(&upper, D * 8);
    add(&lower_f, D * 4);
    add(&upper_f, D * 4);
    add(&boosts, std::max<uint64_t>(v.M, 1) * 8);
    add(&v.pos, F * Dp * 4);
    add(&v.fit, F * 8);
    add(&v.fit_prev, F * 8);
    add(&v.amp, F * 8);
    add(&v.li, F * 8);
    add(&v.improved, F * 4);
    add(&v.winner, F * 4);
    add(&v.loser, F * 4);
    add(&v.pop_lo, c.B * Dp * 4);
    add(&v.pop_hi, c.B * Dp * 4);
    add(&v.sparks, P * Dp * 4);
    if (v.nn) add(&v.sparks_h, P * Dp * 2);
    add(&v.sfit, P * 4);
    add(&v.spart, P * np2 * 4);
    add(&v.rank_idx, std::max<uint64_t>(v.Fl * 2 * v.top, 1) * 4);
    add(&v.guides, std::max<uint64_t>(G, 1) * Dp * 4);
    if (v.nn) add(&v.guides_h, std::max<uint64_t>(G, 1) * Dp * 2);
    add(&v.gfit, std::max<uint64_t>(G, 1) * 4);
    add(&v.gpart, std::max<uint64_t>(G, 1) * np2 * 4);
    if (v.nn) add(&v.fresh_h, F * Dp * 2);
    add(&v.fpart, F * np2 * 4);
    add(&v.best_fit, c.B * 8);
    add(&v.best_pos, c.B * Dp * 4);
    add(&v.best_idx, c.B * 4);
    add(&v.rec_flag, c.B * 4);
    add(&v.tr_evals, trace_cap * c.B * 8);
    add(&v.tr_best, trace_cap * c.B * 8);
    add(&v.tr_ns, trace_cap * c.B * 8);
    add(&v.ctl, sizeof(Ctl));
    if (has_dataset(obj->kind)) {
      add(&X, (size_t)obj->samples * nn_in_dim(obj) * 2);
      add(&y, (size_t)obj->samples * 4);
    }
    size_t total = 0;
    for (auto& s : slots) total += round_up(s.bytes, 256);
    cudaError_t e = cudaMalloc(&arena, total);
    if (e != cudaSuccess) {
      arena = nullptr;
      return Status{MGFWA_ENOMEM, std::string("cudaMalloc(") + std::to_string(total) +
                                      " bytes): " + cudaGetErrorString(e)};
    }
    arena_bytes = total;
    CUDA_TRY(cudaMemset(arena, 0, total));
    size_t off = 0;
    for (auto& s : slots) {
      *s.dst = static_cast<char*>(arena) + off;
      off += round_up(s.bytes, 256);
    }
    v.lower = lower;
    v.upper = upper;
    v.lower_f = lower_f;
    v.upper_f = upper_f;
    v.boosts = boosts;
    STATUS_TRY(configure(c, space, seed));

    if (obj->kind == MGFWA_OBJ_NET) {
      char err[256] = {0};
      auto make = [&](NnPlan& pl, const float* X32, uint64_t rows) -> Status {
        pl.net = net_plan_create(obj->net_id, obj->weight_seed, X32, Dp, rows, err, sizeof err);
        if (!pl.net) return invalid(err);
        return ok();
      };
      STATUS_TRY(make(plan_sparks, v.sparks, P));
      if (G > 0) STATUS_TRY(make(plan_guides, v.guides, G));
      STATUS_TRY(make(plan_fresh, v.pos, F));
    } else if (v.nn) {
      std::vector<__nv_bfloat16> Xh;
      std::vector<int32_t> yh;
      make_dataset(obj->samples, nn_in_dim(obj), nn_out_dim(obj), obj->data_seed, Xh, yh);
      CUDA_TRY(cudaMemcpy(X, Xh.data(), Xh.size() * 2, cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(y, yh.data(), yh.size() * 4, cudaMemcpyHostToDevice));
      char err[256] = {0};
      auto make = [&](NnPlan& pl, const __nv_bfloat16* W, uint64_t rows) -> Status {
        if (obj->kind == MGFWA_OBJ_LENET) {
          pl.lenet = lenet_plan_create(X, y, obj->samples, W, rows, Dp, nsm, err, sizeof err);
          if (!pl.lenet) return invalid(err);
        } else {
          pl.mlp = mlp_plan_create(X, y, obj->samples, obj->in_dim, obj->hidden, obj->out_dim, W,
                                   rows, Dp, nsm, err, sizeof err);
          if (!pl.mlp) return invalid(err);
        }
        return ok();
      };
      STATUS_TRY(make(plan_sparks, v.sparks_h, P));
      if (G > 0) STATUS_TRY(make(plan_guides, v.guides_h, G));
      STATUS_TRY(make(plan_fresh, v.fresh_h, F));
      STATUS_TRY(build_pipeline(obj));
    }
    return ok();
  }
};

// One-entry workspace cache: the device arena, the synthetic dataset and the
// TMA plans of the last destroyed context are kept and handed to the next
// context with the same shape key (the cuFFT-plan / caching-allocator
// pattern), so a repeated run() pays only configure() + initialize().
class WorkspaceCache {
 public:
  static std::unique_ptr<Workspace> take(const std::vector<uint64_t>& key) {
    std::lock_guard<std::mutex> g(mu());
    auto& c = slot();
    if (c && c->key == key) return std::move(c);
    return nullptr;
  }
  static void give(std::unique_ptr<Workspace> w) {
    if (!w) return;
    std::lock_guard<std::mutex> g(mu());
    slot() = std::move(w);  // frees the previous entry
  }
  static void clear() {
    std::lock_guard<std::mutex> g(mu());
    slot().reset();
  }

 private:
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::unique_ptr<Workspace>& slot() {
    // intentionally never destroyed: freeing device memory from a static
    // destructor can run after the CUDA runtime has been torn down
    static auto* s = new std::unique_ptr<Workspace>();
    return *s;
  }
};

// NN fitness hooks used inside the captured generation.
static void hook_sparks(void* p, cudaStream_t s) {
  auto* w = static_cast<Workspace*>(p);
  nn_fitness_launch(w->plan_sparks, w->v.spart, &w->v.ctl->active, s);
}
static void hook_guides(void* p, cudaStream_t s) {
  auto* w = static_cast<Workspace*>(p);
  nn_fitness_launch(w->plan_guides, w->v.gpart, &w->v.ctl->active, s);
}
static void hook_fresh(void* p, cudaStream_t s) {
  auto* w = static_cast<Workspace*>(p);
  nn_fitness_launch(w->plan_fresh, w->v.fpart, &w->v.ctl->n_losers, s);
}
static void hook_fresh_all(void* p, cudaStream_t s) {
  auto* w = static_cast<Workspace*>(p);
  nn_fitness_launch(w->plan_fresh, w->v.fpart, nullptr, s);
}
// Explode of firework chunk c + 1 (auxiliary stream) runs beside the tcgen05
// fitness of chunk c (generation stream): the integer-bound explode fills the
// issue slots the tensor-core kernel leaves idle.  Inside graph capture the
// fork / join events become graph edges.
static void hook_explode_eval(void* p, cudaStream_t s) {
  auto* w = static_cast<Workspace*>(p);
  const EngineView& v = w->v;
  cudaEventRecord(w->ev_fork, s);
  cudaStreamWaitEvent(w->aux, w->ev_fork, 0);
  const size_t G = w->plan_chunks.size();
  launch_explode_fireworks(v, w->chunk_f0[0], w->chunk_nf[0], w->nsm, w->aux);
  cudaEventRecord(w->ev_chunk[0], w->aux);
  for (size_t c = 0; c < G; ++c) {
    cudaStreamWaitEvent(s, w->ev_chunk[c], 0);
    // the next explode chunk is released once every fitness CTA of this
    // chunk is resident (launch-completion edge), so the explode blocks fill
    // the room the persistent tcgen05 CTAs leave instead of taking the SMs first
    mlp_fitness_launch(w->plan_chunks[c].mlp, v.spart + w->chunk_f0[c] * v.lam * v.nparts * 2, &v.ctl->active, s,
                       w->pipe_lc ? w->ev_launched[c] : nullptr);
    if (c + 1 < G) {
      cudaStreamWaitEvent(w->aux, w->pipe_lc ? w->ev_launched[c] : w->ev_chunk[c], 0);
      launch_explode_fireworks(v, w->chunk_f0[c + 1], w->chunk_nf[c + 1], w->nsm, w->aux);
      cudaEventRecord(w->ev_chunk[c + 1], w->aux);
    }
  }
}

// ----------------------------------------------------------------- engine
// NCCL, bound at run time (dlopen "libnccl.so.2": the copy already loaded in
// the process — e.g. PyTorch's — or the system one), so the library has no
// link-time NCCL dependency and single-GPU users never load it.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

static const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllGather && a.AllReduce && a.GroupStart && a.GroupEnd &&
           a.CommDestroy && a.GetErrorString;
    return a;
  }();
  return api;
}

#define NCCL_TRY(expr)                                                                \
  do {                                                                                \
    ncclResult_t r__ = (expr);                                                        \
    if (r__ != ncclSuccess)                                                           \
      return Status{MGFWA_ENCCL, std::string(#expr) + ": " + nccl().GetErrorString(r__)}; \
  } while (0)

class Engine {
 public:
  HostConfig cfg;
  std::unique_ptr<Workspace> ws;
  GenerationHooks hooks{};
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  cudaGraphExec_t gen_exec = nullptr;    // whole loop body (one rank)
  cudaGraphExec_t gen_exec_a = nullptr;  // sharded: up to selection
  cudaGraphExec_t gen_exec_b = nullptr;  // sharded: loser-out .. record
  cudaGraphExec_t gen_exec_ab = nullptr;  // sharded with NCCL: A + captured exchange + B
  uint64_t rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  uint64_t kernels_per_gen = 0;
  Ctl* host_ctl = nullptr;  // pinned
  bool initialized = false;
  std::string last_error;
  // host copy of the trace, [B][wave]
  std::vector<std::vector<uint64_t>> tr_evals;
  std::vector<std::vector<double>> tr_best, tr_wall;
  uint64_t host_trace_n = 0;
  uint64_t pending_gens = 0;  // generations enqueued since the last sync (trace ring bound)
  bool nan_flushed = false;   // replica + NCCL: end-of-run NaN all-reduce done
  std::vector<uint64_t> ring_e;
  std::vector<double> ring_b;
  std::vector<uint64_t> ring_t;

  ~Engine() {
    // gen_exec, own_stream and host_ctl belong to the workspace
    if (gen_exec_a) cudaGraphExecDestroy(gen_exec_a);
    if (gen_exec_b) cudaGraphExecDestroy(gen_exec_b);
    if (gen_exec_ab) cudaGraphExecDestroy(gen_exec_ab);
    if (stream) cudaStreamSynchronize(stream);
    if (own_stream && own_stream != stream) cudaStreamSynchronize(own_stream);
    if (comm) nccl().CommDestroy(comm);
    if (ws) WorkspaceCache::give(std::move(ws));
  }

  Status create(const mgfwa_config_t* c, const mgfwa_space_t* space, const mgfwa_objective_t* obj,
                uint64_t seed, int device, uint64_t shard_rank = 0, uint64_t shard_world = 1) {
    if (c == nullptr) return invalid("MgfwaConfig: null config");
    cfg = to_host(c);
    STATUS_TRY(validate_config(cfg));
    STATUS_TRY(validate_space(space));
    STATUS_TRY(validate_objective(obj, space->dim));
    // engine.cpp:319-323
    if (cfg.max_evals > 0 && cfg.max_evals < cfg.B * cfg.mu)
      return invalid("budget too small: needs at least B * mu evaluations");
    if (shard_world == 0 || shard_rank >= shard_world) return invalid("mgfwa_b200: bad shard rank");
    if (shard_world > 1 && (cfg.max_evals == 0 || cfg.wall_ms > 0.0))
      return invalid(
          "mgfwa_b200: sharded runs need an evaluation budget and no wall-clock budget "
          "(every rank must take the same termination decision)");
    rank = shard_rank;
    world = shard_world;
    ws = WorkspaceCache::take(Workspace::make_key(cfg, space, obj, device, 1024, rank, world));
    if (ws) {
      STATUS_TRY(ws->configure(cfg, space, seed));
    } else {
      ws = std::make_unique<Workspace>();
      STATUS_TRY(ws->build(cfg, space, obj, seed, device, 1024, rank, world));
    }
    ws->v.nan_mode = world > 1 ? 1 : 0;  // 2 once a communicator is attached
    if (!ws->stream) CUDA_TRY(cudaStreamCreateWithFlags(&ws->stream, cudaStreamNonBlocking));
    own_stream = ws->stream;
    stream = own_stream;
    if (!ws->host_ctl) CUDA_TRY(cudaMallocHost(&ws->host_ctl, sizeof(Ctl)));
    host_ctl = ws->host_ctl;
    memset(host_ctl, 0, sizeof(Ctl));
    hooks = GenerationHooks{ws.get(), hook_sparks, hook_guides, hook_fresh, hook_fresh_all,
                            ws->plan_chunks.empty() ? nullptr : hook_explode_eval};
    ring_e.resize(ws->v.trace_cap * cfg.B);
    ring_b.resize(ws->v.trace_cap * cfg.B);
    ring_t.resize(ws->v.trace_cap * cfg.B);
    return ok();
  }

  Status capture_one(int phase, cudaGraphExec_t* out, size_t* nodes) {
    return capture_body([&]() -> Status {
      launch_generation_kernels(ws->v, ws->nsm, own_stream, &hooks, phase);
      return ok();
    }, out, nodes);
  }

  template <typename Body>
  Status capture_body(Body body, cudaGraphExec_t* out, size_t* nodes) {
    cudaGraph_t g = nullptr;
    (void)cudaGetLastError();  // clear a stale error so the check below sees this capture's
    CUDA_TRY(cudaStreamBeginCapture(own_stream, cudaStreamCaptureModeThreadLocal));
    const Status bs = body();
    const cudaError_t le = cudaGetLastError();  // a failed launch inside the capture
    cudaError_t e = cudaStreamEndCapture(own_stream, &g);
    if (bs.code != MGFWA_OK || le != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      if (bs.code != MGFWA_OK) return bs;
      return Status{MGFWA_ECUDA, std::string("kernel launch during graph capture: ") + cudaGetErrorString(le)};
    }
    if (e != cudaSuccess) return Status{MGFWA_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e)};
    cudaGraphGetNodes(g, nullptr, nodes);
    e = cudaGraphInstantiate(out, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return Status{MGFWA_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e)};
    return ok();
  }

  // Sharded stepping (phase A, all-gather, phase B) whenever the context is
  // one of several shards or has a communicator (a 1-rank communicator
  // exercises the exchange path on a single GPU).
  bool sharded() const { return world > 1 || comm != nullptr; }

  // Small analytic problems on one context: the whole loop is one persistent
  // cooperative kernel per enqueue (no graph, no launch per generation).
  bool persistent() const { return !sharded() && small_run_ok(ws->v, ws->nsm); }

  Status capture() {
    if (persistent()) {
      kernels_per_gen = 0;  // one launch per enqueue, any number of generations
      return ok();
    }
    if (!sharded()) {
      if (gen_exec) return ok();
      const unsigned char* vb = reinterpret_cast<const unsigned char*>(&ws->v);
      if (ws->exec_all && ws->exec_view.size() == sizeof(EngineView) &&
          memcmp(ws->exec_view.data(), vb, sizeof(EngineView)) == 0) {
        gen_exec = ws->exec_all;  // same workspace, same kernel arguments
        kernels_per_gen = ws->exec_nodes;
        return ok();
      }
      size_t n = 0;
      cudaGraphExec_t g = nullptr;
      STATUS_TRY(capture_one(kGenAll, &g, &n));
      if (ws->exec_all) cudaGraphExecDestroy(ws->exec_all);
      ws->exec_all = gen_exec = g;
      ws->exec_view.assign(vb, vb + sizeof(EngineView));
      ws->exec_nodes = kernels_per_gen = n;
      return ok();
    }
    if (gen_exec_a || gen_exec_ab) return ok();
    if (comm != nullptr) {
      // One graph per generation: phase A, the NCCL exchange (captured:
      // NCCL >= 2.9 records its kernels into the graph) and phase B — no
      // host round trip between the phases.  Falls back to two graphs with
      // host-enqueued collectives when the capture is refused.
      const char* env = getenv("MGFWA_NCCL_GRAPH");
      if (!(env && env[0] == '0')) {
        size_t n = 0;
        const Status st = capture_body([&]() -> Status {
          launch_generation_kernels(ws->v, ws->nsm, own_stream, &hooks, kGenA);
          STATUS_TRY(exchange_nccl(own_stream));
          launch_generation_kernels(ws->v, ws->nsm, own_stream, &hooks, kGenB);
          return ok();
        }, &gen_exec_ab, &n);
        if (st.code == MGFWA_OK) {
          // count this library's kernels only (the graph also holds NCCL's)
          size_t na = 0, nb = 0;
          cudaGraphExec_t ga = nullptr, gb = nullptr;
          STATUS_TRY(capture_one(kGenA, &ga, &na));
          STATUS_TRY(capture_one(kGenB, &gb, &nb));
          cudaGraphExecDestroy(ga);
          cudaGraphExecDestroy(gb);
          kernels_per_gen = na + nb;
          return ok();
        }
        gen_exec_ab = nullptr;
        (void)cudaGetLastError();
      }
    }
    size_t na = 0, nb = 0;
    STATUS_TRY(capture_one(kGenA, &gen_exec_a, &na));
    STATUS_TRY(capture_one(kGenB, &gen_exec_b, &nb));
    kernels_per_gen = na + nb;
    return ok();
  }

  // ---- firework sharding: the per-generation exchange.
  // After selection every rank holds the new state of its own fireworks;
  // one all-gather (in place) replicates {position row, fitness,
  // amplitude, last improvement} of all F fireworks on every rank.
  Status attach_nccl(const void* unique_id, int nranks, int r) {
    if ((uint64_t)nranks != world || (uint64_t)r != rank)
      return invalid("mgfwa_attach_nccl: rank / world do not match the shard");
    if (!nccl().ok) return Status{MGFWA_ENCCL, "libnccl.so.2 not loadable"};
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof(id));
    CUDA_TRY(cudaSetDevice(ws->device));
    NCCL_TRY(nccl().CommInitRank(&comm, nranks, id, r));
    ws->v.nan_mode = 2;  // NaN counts of shard-local work are all-reduced by the exchange
    return ok();
  }

  // Replica sharding (MGFWA_SHARD_REPLICA): the shards own whole batches,
  // which interact only through the evaluation counter (loser-out adds the
  // losers of every batch), so the exchange is one 8-byte sum.
  Status set_shard_mode(int mode) {
    if (initialized) return Status{MGFWA_ESTATE, "mgfwa_set_shard_mode: call before initialize()"};
    if (mode != MGFWA_SHARD_FIREWORK && mode != MGFWA_SHARD_REPLICA)
      return invalid("mgfwa_set_shard_mode: unknown mode");
    EngineView& v = ws->v;
    if (mode == MGFWA_SHARD_FIREWORK) {
      v.replica = 0, v.b_lo = 0, v.b_hi = v.B;
      return ok();
    }
    if (cfg.B % world != 0)
      return invalid("mgfwa_set_shard_mode: replica sharding needs batches divisible by the number of ranks");
    v.replica = 1;
    v.b_lo = v.f_lo / v.mu;
    v.b_hi = (v.f_lo + v.Fl) / v.mu;
    CUDA_TRY(cudaMemsetAsync(v.loser, 0, v.F * sizeof(int), stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    return ok();
  }

  Status exchange_nccl(cudaStream_t st) {
    const EngineView& v = ws->v;
    NCCL_TRY(nccl().GroupStart());
    NCCL_TRY(nccl().AllReduce(&v.ctl->nan_own, &v.ctl->nan_all, 1, ncclUint64, ncclSum, comm, st));
    if (v.replica) {
      NCCL_TRY(nccl().AllReduce(&v.ctl->n_losers_all, &v.ctl->n_losers_all, 1, ncclUint64, ncclSum, comm,
                                st));
      NCCL_TRY(nccl().GroupEnd());
      return ok();
    }
    const size_t rows = v.Fl * v.Dp;
    NCCL_TRY(nccl().AllGather(v.pos + v.f_lo * v.Dp, v.pos, rows, ncclFloat, comm, st));
    NCCL_TRY(nccl().AllGather(v.fit + v.f_lo, v.fit, v.Fl, ncclFloat64, comm, st));
    NCCL_TRY(nccl().AllGather(v.amp + v.f_lo, v.amp, v.Fl, ncclFloat64, comm, st));
    NCCL_TRY(nccl().AllGather(v.li + v.f_lo, v.li, v.Fl, ncclFloat64, comm, st));
    NCCL_TRY(nccl().GroupEnd());
    return ok();
  }

  // In-process exchange (tests / one-GPU emulation of several shards): copy
  // the owned rows of `src` into this shard's replica.
  Status import_shard(const Engine& src) {
    const EngineView& a = ws->v;
    const EngineView& b = src.ws->v;
    if (a.F != b.F || a.Dp != b.Dp || a.Fl != b.Fl) return invalid("mgfwa_shard_exchange: shape mismatch");
    if (a.replica != b.replica) return invalid("mgfwa_shard_exchange: shard modes differ");
    launch_add_losers(a.ctl, b.ctl, a.replica, stream);
    if (a.replica) {
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaStreamSynchronize(stream));
      return ok();
    }
    CUDA_TRY(cudaMemcpyAsync(a.pos + b.f_lo * a.Dp, b.pos + b.f_lo * b.Dp, b.Fl * b.Dp * 4,
                             cudaMemcpyDeviceToDevice, stream));
    CUDA_TRY(cudaMemcpyAsync(a.fit + b.f_lo, b.fit + b.f_lo, b.Fl * 8, cudaMemcpyDeviceToDevice, stream));
    CUDA_TRY(cudaMemcpyAsync(a.amp + b.f_lo, b.amp + b.f_lo, b.Fl * 8, cudaMemcpyDeviceToDevice, stream));
    CUDA_TRY(cudaMemcpyAsync(a.li + b.f_lo, b.li + b.f_lo, b.Fl * 8, cudaMemcpyDeviceToDevice, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    return ok();
  }

  Status phase(int ph) {
    if (!initialized) return Status{MGFWA_ESTATE, "mgfwa: initialize() must precede the loop"};
    launch_generation_kernels(ws->v, ws->nsm, stream, &hooks, ph);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(stream));
    if (ph == kGenB && ++pending_gens >= ws->v.trace_cap - 2) STATUS_TRY(sync());
    return ok();
  }

  Status initialize() {
    CUDA_TRY(cudaSetDevice(ws->device));
    CUDA_TRY(cudaMemsetAsync(ws->v.ctl, 0, sizeof(Ctl), stream));
    launch_initialize_kernels(ws->v, ws->nsm, stream, &hooks);
    CUDA_TRY(cudaGetLastError());
    tr_evals.assign(cfg.B, {});
    tr_best.assign(cfg.B, {});
    tr_wall.assign(cfg.B, {});
    host_trace_n = 0;
    nan_flushed = false;
    STATUS_TRY(sync());
    initialized = true;
    return capture();
  }

  // D2H of the control block and of the new trace points.
  Status sync() {
    CUDA_TRY(cudaMemcpyAsync(host_ctl, ws->v.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    pending_gens = 0;
    const uint64_t n = host_ctl->trace_n;
    if (n > host_trace_n) {
      const uint64_t cap = ws->v.trace_cap, B = cfg.B;
      CUDA_TRY(cudaMemcpyAsync(ring_e.data(), ws->v.tr_evals, cap * B * 8, cudaMemcpyDeviceToHost, stream));
      CUDA_TRY(cudaMemcpyAsync(ring_b.data(), ws->v.tr_best, cap * B * 8, cudaMemcpyDeviceToHost, stream));
      CUDA_TRY(cudaMemcpyAsync(ring_t.data(), ws->v.tr_ns, cap * B * 8, cudaMemcpyDeviceToHost, stream));
      CUDA_TRY(cudaStreamSynchronize(stream));
      const uint64_t first = n > cap && host_trace_n < n - cap ? n - cap : host_trace_n;
      for (uint64_t w = first; w < n; ++w) {
        const uint64_t slot = w % cap;
        for (uint64_t b = 0; b < B; ++b) {
          tr_evals[b].push_back(ring_e[slot * B + b]);
          tr_best[b].push_back(ring_b[slot * B + b]);
          tr_wall[b].push_back((double)ring_t[slot * B + b] * 1e-6);
        }
      }
      host_trace_n = n;
    }
    return ok();
  }

  // The device trace is a ring of trace_cap waves; at most trace_cap - 2
  // generations may run between two syncs or the oldest points would be
  // overwritten before the host copies them.  enqueue() syncs internally
  // when a request would cross that bound (so a long asynchronous enqueue
  // becomes partly synchronous instead of losing trace points).
  Status enqueue(uint64_t n) {
    if (!initialized) return Status{MGFWA_ESTATE, "mgfwa: initialize() must precede the loop"};
    const uint64_t room = ws->v.trace_cap - 2;
    while (n > 0) {
      if (pending_gens >= room) STATUS_TRY(sync());
      const uint64_t k = std::min(n, room - pending_gens);
      STATUS_TRY(enqueue_chunk(k));
      pending_gens += k;
      n -= k;
    }
    return ok();
  }

  Status enqueue_chunk(uint64_t n) {
    if (persistent()) {
      if (n > 0) CUDA_TRY(launch_small_run(ws->v, n, stream));
      return ok();
    }
    if (!sharded()) {
      for (uint64_t i = 0; i < n; ++i) CUDA_TRY(cudaGraphLaunch(gen_exec, stream));
      return ok();
    }
    STATUS_TRY(capture());
    if (comm == nullptr)
      return Status{MGFWA_ESTATE, "mgfwa: sharded context needs mgfwa_attach_nccl (or phases + exchange)"};
    for (uint64_t i = 0; i < n; ++i) {
      if (gen_exec_ab) {
        CUDA_TRY(cudaGraphLaunch(gen_exec_ab, stream));
        continue;
      }
      CUDA_TRY(cudaGraphLaunch(gen_exec_a, stream));
      STATUS_TRY(exchange_nccl(stream));
      CUDA_TRY(cudaGraphLaunch(gen_exec_b, stream));
    }
    return ok();
  }

  uint64_t chunk_limit() const {
    const uint64_t cap = std::min<uint64_t>(64, ws->v.trace_cap - 2);
    if (cfg.max_evals > 0) {
      const uint64_t used = host_ctl->used;
      const uint64_t left = cfg.max_evals > used ? cfg.max_evals - used : 0;
      const uint64_t ub = (left + cfg.wave() - 1) / cfg.wave();
      return std::max<uint64_t>(1, std::min(cap, ub));
    }
    return 4;
  }

  Status step(uint64_t max_gens, uint64_t* ran) {
    if (!initialized) return Status{MGFWA_ESTATE, "mgfwa: initialize() must precede the loop"};
    CUDA_TRY(cudaSetDevice(ws->device));
    uint64_t done = 0;
    while (done < max_gens && host_ctl->active) {
      const uint64_t before = host_ctl->gens_run;
      const uint64_t n = std::min(max_gens - done, chunk_limit());
      STATUS_TRY(enqueue(n));
      STATUS_TRY(sync());
      done += host_ctl->gens_run - before;
      if (host_ctl->gens_run == before) break;
    }
    // Replica shards count their own losers' NaN evaluations after the
    // exchange, so the last generation's travel with one more all-reduce.
    if (comm && ws->v.replica && !host_ctl->active && !nan_flushed) {  // collective: every rank ends together
      NCCL_TRY(nccl().AllReduce(&ws->v.ctl->nan_own, &ws->v.ctl->nan_all, 1, ncclUint64, ncclSum, comm, stream));
      launch_fold_nan(ws->v.ctl, stream);
      CUDA_TRY(cudaGetLastError());
      nan_flushed = true;
      STATUS_TRY(sync());
    }
    if (ran) *ran = done;
    return ok();
  }

  Status run(mgfwa_counters_t* out) {
    STATUS_TRY(initialize());
    uint64_t ran = 0;
    STATUS_TRY(step(std::numeric_limits<uint64_t>::max(), &ran));
    if (out) counters(out);
    return ok();
  }

  void counters(mgfwa_counters_t* out) const {
    out->evaluations_used = host_ctl->used;
    out->iterations = host_ctl->gens_run;
    out->losers_reinitialized = host_ctl->losers_total;
    out->nan_evaluations = host_ctl->nan_count;
    out->trace_waves = host_trace_n;
  }

  Status best(double* fit, double* pos) {
    const uint64_t B = cfg.B, D = ws->v.D, Dp = ws->v.Dp;
    std::vector<double> bf(B);
    std::vector<float> bp(B * Dp);
    CUDA_TRY(cudaMemcpyAsync(bf.data(), ws->v.best_fit, B * 8, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaMemcpyAsync(bp.data(), ws->v.best_pos, B * Dp * 4, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    for (uint64_t b = 0; b < B; ++b) {
      if (fit) fit[b] = bf[b];
      if (pos)
        for (uint64_t d = 0; d < D; ++d) pos[b * D + d] = bp[b * Dp + d];
    }
    return ok();
  }

  Status state(double* pos, double* fit, double* amp, double* li) {
    const uint64_t F = ws->v.F, D = ws->v.D, Dp = ws->v.Dp;
    std::vector<float> p(F * Dp);
    std::vector<double> f(F), a(F), l(F);
    CUDA_TRY(cudaMemcpyAsync(p.data(), ws->v.pos, F * Dp * 4, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaMemcpyAsync(f.data(), ws->v.fit, F * 8, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaMemcpyAsync(a.data(), ws->v.amp, F * 8, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaMemcpyAsync(l.data(), ws->v.li, F * 8, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    for (uint64_t i = 0; i < F; ++i) {
      if (pos)
        for (uint64_t d = 0; d < D; ++d) pos[i * D + d] = p[i * Dp + d];
      if (fit) fit[i] = f[i];
      if (amp) amp[i] = a[i];
      if (li) li[i] = l[i];
    }
    return ok();
  }

  // The candidate buffers of the last generation (owned fireworks).
  Status candidates(double* sparks, double* sfit, double* guides, double* gfit, uint16_t* sparks_bf16) {
    const EngineView& v = ws->v;
    const uint64_t P = v.Fl * v.lam, G = v.Fl * v.M, D = v.D, Dp = v.Dp;
    if (sparks_bf16 && v.sparks_h == nullptr)
      return invalid("mgfwa_get_candidates: no bf16 spark shadow (objective is not a tensor-core one)");
    if ((guides || gfit) && G == 0) return invalid("mgfwa_get_candidates: no guiding sparks (M = 0)");
    CUDA_TRY(cudaStreamSynchronize(stream));
    const uint64_t chunk = 4096;  // rows per staging copy (bounded host memory at C5 shapes)
    std::vector<float> rows;
    std::vector<uint16_t> rows_h;
    auto copy_rows = [&](const float* src, uint64_t n, double* dst) -> Status {
      for (uint64_t r0 = 0; r0 < n; r0 += chunk) {
        const uint64_t m = std::min(chunk, n - r0);
        rows.resize(m * Dp);
        CUDA_TRY(cudaMemcpy(rows.data(), src + r0 * Dp, m * Dp * 4, cudaMemcpyDeviceToHost));
        for (uint64_t r = 0; r < m; ++r)
          for (uint64_t d = 0; d < D; ++d) dst[(r0 + r) * D + d] = rows[r * Dp + d];
      }
      return ok();
    };
    auto copy_fit = [&](const float* src, uint64_t n, double* dst) -> Status {
      std::vector<float> f(n);
      CUDA_TRY(cudaMemcpy(f.data(), src, n * 4, cudaMemcpyDeviceToHost));
      for (uint64_t i = 0; i < n; ++i) dst[i] = f[i];
      return ok();
    };
    if (sparks) STATUS_TRY(copy_rows(v.sparks, P, sparks));
    if (sfit) STATUS_TRY(copy_fit(v.sfit, P, sfit));
    if (guides) STATUS_TRY(copy_rows(v.guides, G, guides));
    if (gfit) STATUS_TRY(copy_fit(v.gfit, G, gfit));
    if (sparks_bf16) {
      for (uint64_t r0 = 0; r0 < P; r0 += chunk) {
        const uint64_t m = std::min(chunk, P - r0);
        rows_h.resize(m * Dp);
        CUDA_TRY(cudaMemcpy(rows_h.data(), v.sparks_h + r0 * Dp, m * Dp * 2, cudaMemcpyDeviceToHost));
        for (uint64_t r = 0; r < m; ++r)
          for (uint64_t d = 0; d < D; ++d) sparks_bf16[(r0 + r) * D + d] = rows_h[r * Dp + d];
      }
    }
    return ok();
  }
};

// ------------------------------------------------------- operator helpers
// Host fp64 [rows][D] <-> device fp32 [rows][Dp].
static Status upload_rows(float* dst, const double* src, uint64_t rows, uint64_t D, uint64_t Dp,
                          cudaStream_t s) {
  std::vector<float> h(rows * Dp, 0.0f);
  for (uint64_t r = 0; r < rows; ++r)
    for (uint64_t d = 0; d < D; ++d) h[r * Dp + d] = (float)src[r * D + d];
  CUDA_TRY(cudaMemcpyAsync(dst, h.data(), h.size() * 4, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return ok();
}
static Status download_rows(double* dst, const float* src, uint64_t rows, uint64_t D, uint64_t Dp,
                            cudaStream_t s) {
  std::vector<float> h(rows * Dp);
  CUDA_TRY(cudaMemcpyAsync(h.data(), src, h.size() * 4, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  for (uint64_t r = 0; r < rows; ++r)
    for (uint64_t d = 0; d < D; ++d) dst[r * D + d] = (double)h[r * Dp + d];
  return ok();
}
template <typename T>
static Status upload(T* dst, const T* src, uint64_t n, cudaStream_t s) {
  CUDA_TRY(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return ok();
}
template <typename T>
static Status download(T* dst, const T* src, uint64_t n, cudaStream_t s) {
  CUDA_TRY(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return ok();
}

// A workspace for operator seams: an analytic objective unless given.
static Status op_workspace(std::unique_ptr<Workspace>& ws, const HostConfig& c,
                           const mgfwa_space_t* space, const mgfwa_objective_t* obj) {
  mgfwa_objective_t sphere{MGFWA_OBJ_SPHERE, 0, 0, 0, 0, 0};
  ws = std::make_unique<Workspace>();
  STATUS_TRY(ws->build(c, space, obj ? obj : &sphere, 0, 0, 4));
  return ok();
}

static Status set_ctl(Workspace& w, uint64_t iteration, uint64_t used, int active) {
  Ctl c{};
  c.iteration = iteration;
  c.used = used;
  c.active = active;
  CUDA_TRY(cudaMemcpy(w.v.ctl, &c, sizeof(Ctl), cudaMemcpyHostToDevice));
  return ok();
}

static mgfwa_space_t wide_space(uint64_t D, std::vector<double>& lo, std::vector<double>& hi) {
  lo.assign(D, -3.0e38);
  hi.assign(D, 3.0e38);
  return mgfwa_space_t{lo.data(), hi.data(), D};
}

static HostConfig relaxed(const mgfwa_config_t* c) {
  HostConfig h = to_host(c);
  if (h.max_evals == 0 && !(h.wall_ms > 0.0)) h.max_evals = 1ull << 62;
  return h;
}

}  // namespace mgfwa_b200

// ===================================================================== C-ABI
using namespace mgfwa_b200;

struct mgfwa_ctx {
  Engine engine;
};

static int fail(mgfwa_ctx* ctx, const Status& s) {
  if (s.code == MGFWA_OK) return MGFWA_OK;
  if (ctx) ctx->engine.last_error = s.msg;
  g_last_error = s.msg;
  return s.code;
}

extern "C" {

const char* mgfwa_version(void) { return "mgfwa_b200 0.2 (sm_100a)"; }

int mgfwa_release_cached_workspace(void) {
  WorkspaceCache::clear();
  return MGFWA_OK;
}

const char* mgfwa_last_error(mgfwa_ctx_t ctx) {
  return ctx ? ctx->engine.last_error.c_str() : g_last_error.c_str();
}

int mgfwa_create(const mgfwa_config_t* config, const mgfwa_space_t* space,
                 const mgfwa_objective_t* objective, uint64_t seed, int device, mgfwa_ctx_t* out) {
  if (!out) return fail(nullptr, invalid("mgfwa_create: null output"));
  *out = nullptr;
  auto* ctx = new (std::nothrow) mgfwa_ctx();
  if (!ctx) return fail(nullptr, Status{MGFWA_ENOMEM, "host allocation"});
  Status s = ctx->engine.create(config, space, objective, seed, device);
  if (s.code != MGFWA_OK) {
    fail(nullptr, s);
    delete ctx;
    return s.code;
  }
  *out = ctx;
  return MGFWA_OK;
}

int mgfwa_destroy(mgfwa_ctx_t ctx) {
  delete ctx;
  return MGFWA_OK;
}

int mgfwa_create_shard(const mgfwa_config_t* config, const mgfwa_space_t* space,
                       const mgfwa_objective_t* objective, uint64_t seed, int device, int rank,
                       int world, mgfwa_ctx_t* out) {
  if (!out) return fail(nullptr, invalid("mgfwa_create_shard: null output"));
  *out = nullptr;
  if (rank < 0 || world < 1) return fail(nullptr, invalid("mgfwa_b200: bad shard rank"));
  auto* ctx = new (std::nothrow) mgfwa_ctx();
  if (!ctx) return fail(nullptr, Status{MGFWA_ENOMEM, "host allocation"});
  Status s = ctx->engine.create(config, space, objective, seed, device, (uint64_t)rank,
                                (uint64_t)world);
  if (s.code != MGFWA_OK) {
    fail(nullptr, s);
    delete ctx;
    return s.code;
  }
  *out = ctx;
  return MGFWA_OK;
}

int mgfwa_nccl_unique_id(void* out128) {
  if (!nccl().ok) return fail(nullptr, Status{MGFWA_ENCCL, "libnccl.so.2 not loadable"});
  ncclUniqueId id;
  const ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, Status{MGFWA_ENCCL, nccl().GetErrorString(r)});
  memcpy(out128, &id, sizeof(id));
  return MGFWA_OK;
}

int mgfwa_attach_nccl(mgfwa_ctx_t ctx, const void* unique_id128, int nranks, int rank) {
  return fail(ctx, ctx->engine.attach_nccl(unique_id128, nranks, rank));
}

int mgfwa_generation_phase(mgfwa_ctx_t ctx, int phase) {
  if (phase != 1 && phase != 2) return fail(ctx, invalid("mgfwa_generation_phase: phase is 1 or 2"));
  Status s = ctx->engine.phase(phase == 1 ? kGenA : kGenB);
  if (s.code == MGFWA_OK && phase == 2) s = ctx->engine.sync();
  return fail(ctx, s);
}

int mgfwa_set_shard_mode(mgfwa_ctx_t ctx, int mode) { return fail(ctx, ctx->engine.set_shard_mode(mode)); }

int mgfwa_shard_exchange(mgfwa_ctx_t dst, mgfwa_ctx_t src) {
  return fail(dst, dst->engine.import_shard(src->engine));
}

int mgfwa_set_stream(mgfwa_ctx_t ctx, void* s) {
  ctx->engine.stream = s ? static_cast<cudaStream_t>(s) : ctx->engine.own_stream;
  return MGFWA_OK;
}

int mgfwa_kernels_per_generation(mgfwa_ctx_t ctx, uint64_t* n) {
  Status s = ctx->engine.capture();
  if (s.code) return fail(ctx, s);
  *n = ctx->engine.kernels_per_gen;
  return MGFWA_OK;
}

int mgfwa_initialize(mgfwa_ctx_t ctx) { return fail(ctx, ctx->engine.initialize()); }

int mgfwa_step(mgfwa_ctx_t ctx, uint64_t max_generations, uint64_t* generations_run) {
  return fail(ctx, ctx->engine.step(max_generations, generations_run));
}

int mgfwa_enqueue_generations(mgfwa_ctx_t ctx, uint64_t n) { return fail(ctx, ctx->engine.enqueue(n)); }

int mgfwa_sync(mgfwa_ctx_t ctx) { return fail(ctx, ctx->engine.sync()); }

int mgfwa_run(mgfwa_ctx_t ctx, mgfwa_counters_t* counters) {
  return fail(ctx, ctx->engine.run(counters));
}

int mgfwa_get_counters(mgfwa_ctx_t ctx, mgfwa_counters_t* out) {
  ctx->engine.counters(out);
  return MGFWA_OK;
}

int mgfwa_get_best(mgfwa_ctx_t ctx, double* best_fitness, double* best_position) {
  return fail(ctx, ctx->engine.best(best_fitness, best_position));
}

int mgfwa_get_trace(mgfwa_ctx_t ctx, uint64_t* evaluations, double* best, double* wall_ms,
                    uint64_t cap, uint64_t* waves) {
  Engine& e = ctx->engine;
  const uint64_t n = e.host_trace_n;
  if (waves) *waves = n;
  for (uint64_t b = 0; b < e.cfg.B; ++b)
    for (uint64_t w = 0; w < n && w < cap && w < e.tr_evals[b].size(); ++w) {
      if (evaluations) evaluations[b * cap + w] = e.tr_evals[b][w];
      if (best) best[b * cap + w] = e.tr_best[b][w];
      if (wall_ms) wall_ms[b * cap + w] = e.tr_wall[b][w];
    }
  return MGFWA_OK;
}

int mgfwa_get_state(mgfwa_ctx_t ctx, double* positions, double* fitness, double* amplitudes,
                    double* last_improvement) {
  return fail(ctx, ctx->engine.state(positions, fitness, amplitudes, last_improvement));
}

int mgfwa_get_candidates(mgfwa_ctx_t ctx, double* sparks, double* spark_fitness, double* guides,
                         double* guide_fitness, uint16_t* sparks_bf16) {
  return fail(ctx, ctx->engine.candidates(sparks, spark_fitness, guides, guide_fitness, sparks_bf16));
}

int mgfwa_run_once(const mgfwa_config_t* config, const mgfwa_space_t* space,
                   const mgfwa_objective_t* objective, uint64_t seed, int device,
                   double* best_fitness, double* best_position, uint64_t* trace_evaluations,
                   double* trace_best, double* trace_wall_ms, uint64_t trace_cap,
                   mgfwa_counters_t* counters) {
  mgfwa_ctx_t ctx = nullptr;
  int rc = mgfwa_create(config, space, objective, seed, device, &ctx);
  if (rc) return rc;
  rc = mgfwa_run(ctx, counters);
  if (!rc) rc = mgfwa_get_best(ctx, best_fitness, best_position);
  if (!rc && (trace_evaluations || trace_best || trace_wall_ms))
    rc = mgfwa_get_trace(ctx, trace_evaluations, trace_best, trace_wall_ms, trace_cap, nullptr);
  if (rc) g_last_error = ctx->engine.last_error;
  mgfwa_destroy(ctx);
  return rc;
}

// ------------------------------------------------------------------ ops
int mgfwa_op_initialize(const mgfwa_config_t* config, const mgfwa_space_t* space,
                        const mgfwa_objective_t* objective, uint64_t seed, double* positions,
                        double* fitness, double* amplitudes) {
  mgfwa_ctx_t ctx = nullptr;
  mgfwa_config_t c = *config;
  if (c.max_evaluations == 0 && !(c.wall_clock_budget_ms > 0)) c.max_evaluations = 1ull << 62;
  int rc = mgfwa_create(&c, space, objective, seed, 0, &ctx);
  if (rc) return rc;
  rc = mgfwa_initialize(ctx);
  if (!rc) rc = mgfwa_get_state(ctx, positions, fitness, amplitudes, nullptr);
  if (rc) g_last_error = ctx->engine.last_error;
  mgfwa_destroy(ctx);
  return rc;
}

int mgfwa_op_explode_map(const mgfwa_config_t* config, const mgfwa_space_t* space,
                         const double* positions, const double* amplitudes, uint64_t iteration,
                         uint64_t seed, double* sparks) {
  auto body = [&]() -> Status {
    HostConfig c = relaxed(config);
    STATUS_TRY(validate_space(space));
    std::unique_ptr<Workspace> w;
    STATUS_TRY(op_workspace(w, c, space, nullptr));
    EngineView v = w->v;
    v.seed = seed;
    cudaStream_t s = 0;
    STATUS_TRY(upload_rows(v.pos, positions, v.F, v.D, v.Dp, s));
    STATUS_TRY(upload(v.amp, amplitudes, v.F, s));
    STATUS_TRY(set_ctl(*w, iteration, 0, 1));
    launch_pop_range(v, w->nsm, s);
    launch_explode_map(v, w->nsm, s);
    CUDA_TRY(cudaGetLastError());
    return download_rows(sparks, v.sparks, v.F * v.lam, v.D, v.Dp, s);
  };
  return fail(nullptr, body());
}

int mgfwa_op_random_mapping(const mgfwa_space_t* space, const double* cand, uint64_t B,
                            uint64_t rows, uint64_t per, const double* positions, uint64_t mu,
                            uint64_t iteration, uint64_t seed, uint64_t stream, double* out) {
  auto body = [&]() -> Status {
    STATUS_TRY(validate_space(space));
    HostConfig c;
    c.B = B;
    c.mu = mu;
    c.lam = 2 * rows;  // sparks buffer holds the candidates and the output
    c.M = 0;
    c.max_evals = 1;
    std::unique_ptr<Workspace> w;
    STATUS_TRY(op_workspace(w, c, space, nullptr));
    EngineView v = w->v;
    v.seed = seed;
    // the candidate cube is B x rows; stage it in the (F*lam >= B*rows) sparks buffer
    cudaStream_t s = 0;
    STATUS_TRY(upload_rows(v.pos, positions, v.F, v.D, v.Dp, s));
    STATUS_TRY(upload_rows(v.sparks, cand, B * rows, v.D, v.Dp, s));
    STATUS_TRY(set_ctl(*w, iteration, 0, 1));
    launch_pop_range(v, w->nsm, s);
    float* outd = v.sparks + B * rows * v.Dp;  // second half of the buffer (F*lam >= 2*B*rows)
    if (v.F * v.lam < 2 * B * rows) return invalid("random_mapping: internal sizing");
    launch_map_rows(v, v.sparks, outd, rows, per, stream, iteration, s);
    CUDA_TRY(cudaGetLastError());
    return download_rows(out, outd, B * rows, v.D, v.Dp, s);
  };
  return fail(nullptr, body());
}

int mgfwa_op_guides(const mgfwa_config_t* config, const mgfwa_space_t* space,
                    const double* positions, const double* sparks, const double* spark_fitness,
                    uint64_t iteration, uint64_t seed, double* guides) {
  auto body = [&]() -> Status {
    HostConfig c = relaxed(config);
    STATUS_TRY(validate_config(c));
    STATUS_TRY(validate_space(space));
    if (c.M == 0) return invalid("guides: M must be positive");
    std::unique_ptr<Workspace> w;
    STATUS_TRY(op_workspace(w, c, space, nullptr));
    EngineView v = w->v;
    v.seed = seed;
    v.injected_fitness = 1;
    cudaStream_t s = 0;
    STATUS_TRY(upload_rows(v.pos, positions, v.F, v.D, v.Dp, s));
    STATUS_TRY(upload_rows(v.sparks, sparks, v.F * v.lam, v.D, v.Dp, s));
    std::vector<float> sf(v.F * v.lam);
    for (uint64_t i = 0; i < sf.size(); ++i) sf[i] = (float)spark_fitness[i];
    STATUS_TRY(upload(v.sfit, sf.data(), sf.size(), s));
    STATUS_TRY(set_ctl(*w, iteration, 0, 1));
    launch_pop_range(v, w->nsm, s);
    launch_rank(v, s);
    launch_guides(v, w->nsm, s);
    CUDA_TRY(cudaGetLastError());
    return download_rows(guides, v.guides, v.F * v.M, v.D, v.Dp, s);
  };
  return fail(nullptr, body());
}

int mgfwa_op_guiding_vector(const mgfwa_config_t* config, uint64_t dim, const double* sparks,
                            const double* spark_fitness, double* delta) {
  // guiding_vector through the production kernels: pos = 0, one guide with
  // beta = 1 and an unbounded box, so guide = 0 + 1 * delta exactly.
  auto body = [&]() -> Status {
    HostConfig c = relaxed(config);
    if (c.lam < 2 * c.top()) return invalid("guiding_vector: elite and poor sets overlap");
    c.M = 1;
    c.boosts = {1.0};
    std::vector<double> lo, hi;
    mgfwa_space_t sp = wide_space(dim, lo, hi);
    std::unique_ptr<Workspace> w;
    STATUS_TRY(op_workspace(w, c, &sp, nullptr));
    EngineView v = w->v;
    v.injected_fitness = 1;
    cudaStream_t s = 0;
    STATUS_TRY(upload_rows(v.sparks, sparks, v.F * v.lam, v.D, v.Dp, s));
    std::vector<float> sf(v.F * v.lam);
    for (uint64_t i = 0; i < sf.size(); ++i) sf[i] = (float)spark_fitness[i];
    STATUS_TRY(upload(v.sfit, sf.data(), sf.size(), s));
    STATUS_TRY(set_ctl(*w, 1, 0, 1));
    launch_rank(v, s);
    launch_guides(v, w->nsm, s);
    CUDA_TRY(cudaGetLastError());
    return download_rows(delta, v.guides, v.F, v.D, v.Dp, s);
  };
  return fail(nullptr, body());
}

int mgfwa_op_select_best(const mgfwa_config_t* config, const mgfwa_space_t* space,
                         const double* positions, const double* fitness, const double* amplitudes,
                         const double* sparks, const double* spark_fitness, const double* guides,
                         const double* guide_fitness, double* new_positions, double* new_fitness,
                         double* new_last_improvement, double* improved, double* new_amplitudes) {
  auto body = [&]() -> Status {
    HostConfig c = relaxed(config);
    STATUS_TRY(validate_space(space));
    if (guides == nullptr) c.M = 0, c.boosts.clear();
    std::unique_ptr<Workspace> w;
    STATUS_TRY(op_workspace(w, c, space, nullptr));
    EngineView v = w->v;
    v.injected_fitness = 1;
    cudaStream_t s = 0;
    STATUS_TRY(upload_rows(v.pos, positions, v.F, v.D, v.Dp, s));
    STATUS_TRY(upload(v.fit, fitness, v.F, s));
    STATUS_TRY(upload(v.amp, amplitudes, v.F, s));
    STATUS_TRY(upload_rows(v.sparks, sparks, v.F * v.lam, v.D, v.Dp, s));
    std::vector<float> sf(v.F * v.lam);
    for (uint64_t i = 0; i < sf.size(); ++i) sf[i] = (float)spark_fitness[i];
    STATUS_TRY(upload(v.sfit, sf.data(), sf.size(), s));
    if (v.M > 0) {
      STATUS_TRY(upload_rows(v.guides, guides, v.F * v.M, v.D, v.Dp, s));
      std::vector<float> gf(v.F * v.M);
      for (uint64_t i = 0; i < gf.size(); ++i) gf[i] = (float)guide_fitness[i];
      STATUS_TRY(upload(v.gfit, gf.data(), gf.size(), s));
    }
    STATUS_TRY(set_ctl(*w, 1, 0, 1));
    launch_select(v, w->nsm, s);
    CUDA_TRY(cudaGetLastError());
    STATUS_TRY(download_rows(new_positions, v.pos, v.F, v.D, v.Dp, s));
    STATUS_TRY(download(new_fitness, v.fit, v.F, s));
    STATUS_TRY(download(new_last_improvement, v.li, v.F, s));
    std::vector<int> imp(v.F);
    STATUS_TRY(download(imp.data(), v.improved, v.F, s));
    for (uint64_t i = 0; i < v.F; ++i) improved[i] = imp[i] ? 1.0 : 0.0;
    if (new_amplitudes) STATUS_TRY(download(new_amplitudes, v.amp, v.F, s));
    return ok();
  };
  return fail(nullptr, body());
}

int mgfwa_op_loser_out(const mgfwa_config_t* config, const mgfwa_space_t* space,
                       const mgfwa_objective_t* objective, double* positions, double* fitness,
                       double* amplitudes, double* last_improvement, uint64_t* used,
                       uint64_t iteration, uint64_t seed, double iterations_remaining,
                       uint64_t* reinit) {
  auto body = [&]() -> Status {
    HostConfig c = relaxed(config);
    STATUS_TRY(validate_space(space));
    STATUS_TRY(validate_objective(objective, space->dim));
    std::unique_ptr<Workspace> w;
    STATUS_TRY(op_workspace(w, c, space, objective));
    EngineView v = w->v;
    v.seed = seed;
    v.has_iters_override = 1;
    v.iters_override = iterations_remaining;
    v.max_evals = 0;
    v.wall_budget_ms = 0;
    cudaStream_t s = 0;
    STATUS_TRY(upload_rows(v.pos, positions, v.F, v.D, v.Dp, s));
    STATUS_TRY(upload(v.fit, fitness, v.F, s));
    STATUS_TRY(upload(v.amp, amplitudes, v.F, s));
    STATUS_TRY(upload(v.li, last_improvement, v.F, s));
    STATUS_TRY(set_ctl(*w, iteration, *used, 1));
    launch_loser(v, w->nsm, s);
    if (v.nn) {
      w->v = v;
      hook_fresh(w.get(), s);
    }
    launch_loser_commit(v, w->nsm, s);
    CUDA_TRY(cudaGetLastError());
    STATUS_TRY(download_rows(positions, v.pos, v.F, v.D, v.Dp, s));
    STATUS_TRY(download(fitness, v.fit, v.F, s));
    STATUS_TRY(download(amplitudes, v.amp, v.F, s));
    STATUS_TRY(download(last_improvement, v.li, v.F, s));
    Ctl ctl;
    STATUS_TRY(download(&ctl, v.ctl, 1, s));
    *reinit = (uint64_t)ctl.n_losers;
    *used = ctl.used;
    return ok();
  };
  return fail(nullptr, body());
}

int mgfwa_op_batched_apply(const mgfwa_objective_t* objective, const double* rows, uint64_t n,
                           uint64_t dim, double* fitness, uint64_t* nan_count) {
  auto body = [&]() -> Status {
    STATUS_TRY(validate_objective(objective, dim));
    HostConfig c;
    c.B = 1;
    c.mu = n;
    c.lam = 1;
    c.M = 0;
    c.max_evals = 1ull << 62;
    std::vector<double> lo, hi;
    mgfwa_space_t sp = wide_space(dim, lo, hi);
    std::unique_ptr<Workspace> w;
    STATUS_TRY(op_workspace(w, c, &sp, objective));
    EngineView v = w->v;
    cudaStream_t s = 0;
    STATUS_TRY(upload_rows(v.pos, rows, n, dim, v.Dp, s));
    if (v.nn) {
      launch_to_bf16(v.pos, v.fresh_h, n * v.Dp, s);
      hook_fresh_all(w.get(), s);
    } else {
      launch_analytic_partials(v.pos, n, dim, v.Dp, v.nch, v.obj_kind, v.fpart, w->nsm, s);
    }
    unsigned long long* dnan = reinterpret_cast<unsigned long long*>(&v.ctl->nan_count);
    launch_finalize_rows(v, v.fpart, n, v.sfit, dnan, s);
    CUDA_TRY(cudaGetLastError());
    std::vector<float> f(n);
    STATUS_TRY(download(f.data(), v.sfit, n, s));
    for (uint64_t i = 0; i < n; ++i) fitness[i] = (double)f[i];
    Ctl ctl;
    STATUS_TRY(download(&ctl, v.ctl, 1, s));
    if (nan_count) *nan_count = ctl.nan_count;
    return ok();
  };
  return fail(nullptr, body());
}

int mgfwa_op_argmin_per_population(const double* fitness, uint64_t rows, uint64_t cols,
                                   uint64_t* index, double* value) {
  auto body = [&]() -> Status {
    double* df = nullptr;
    uint64_t* di = nullptr;
    double* dv = nullptr;
    CUDA_TRY(cudaMalloc(&df, rows * cols * 8));
    CUDA_TRY(cudaMalloc(&di, rows * 8));
    CUDA_TRY(cudaMalloc(&dv, rows * 8));
    CUDA_TRY(cudaMemcpy(df, fitness, rows * cols * 8, cudaMemcpyHostToDevice));
    launch_argmin_rows(df, rows, cols, di, dv, 0);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpy(index, di, rows * 8, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(value, dv, rows * 8, cudaMemcpyDeviceToHost));
    cudaFree(df);
    cudaFree(di);
    cudaFree(dv);
    return ok();
  };
  return fail(nullptr, body());
}

// L2 flush for cold-cache kernel timing: write 256 MB (twice the L2).
static cudaError_t flush_l2(cudaStream_t s) {
  static void* buf = nullptr;
  constexpr size_t kBytes = 256ull << 20;
  if (buf == nullptr) {
    cudaError_t r = cudaMalloc(&buf, kBytes);
    if (r != cudaSuccess) return r;
  }
  return cudaMemsetAsync(buf, 0x5a, kBytes, s);
}

int mgfwa_time_kernel(mgfwa_ctx_t ctx, int kernel, uint64_t iters, double* ms, uint64_t* units) {
  Engine& e = ctx->engine;
  auto body = [&]() -> Status {
    if (!e.initialized) return Status{MGFWA_ESTATE, "mgfwa: initialize() must precede timing"};
    Workspace& w = *e.ws;
    const EngineView& v = w.v;
    std::function<void()> launch;
    switch (kernel) {
      case MGFWA_KERNEL_FITNESS:  // the dominant kernel of the workload
        if (v.nn)
          launch = [&]() { nn_fitness_launch(w.plan_sparks, v.spart, nullptr, e.stream); };
        else
          launch = [&]() { launch_explode_map(v, w.nsm, e.stream); };
        *units = v.Fl * v.lam;
        break;
      case MGFWA_KERNEL_EXPLODE:
        launch = [&]() { launch_explode_map(v, w.nsm, e.stream); };
        *units = v.Fl * v.lam;
        break;
      case MGFWA_KERNEL_RANK:
        launch = [&]() { launch_rank(v, e.stream); };
        *units = v.Fl * v.lam;
        break;
      case MGFWA_KERNEL_GUIDES:
        if (v.M == 0) return invalid("mgfwa_time_kernel: no guides");
        launch = [&]() { launch_guides(v, w.nsm, e.stream); };
        *units = v.Fl * v.M;
        break;
      case MGFWA_KERNEL_GUIDE_FITNESS:
        if (v.M == 0 || !v.nn) return invalid("mgfwa_time_kernel: no NN guide fitness");
        launch = [&]() { nn_fitness_launch(w.plan_guides, v.gpart, nullptr, e.stream); };
        *units = v.Fl * v.M;
        break;
      case MGFWA_KERNEL_SELECT: {
        // not state-idempotent: the state k_select writes is snapshotted and
        // restored (untimed) before every timed launch and at the end
        const size_t pos_b = v.F * v.Dp * 4, f8 = v.F * 8, f4 = v.F * 4, g4 = v.F * (v.M ? v.M : 1) * 4;
        std::vector<std::pair<void*, size_t>> st = {{v.pos, pos_b}, {v.fit, f8}, {v.amp, f8}, {v.li, f8},
                                                    {v.improved, f4}, {v.winner, f4}, {v.gfit, g4},
                                                    {v.ctl, sizeof(Ctl)}};
        size_t total = 0;
        for (auto& x : st) total += (x.second + 255) & ~size_t(255);
        char* snap = nullptr;
        CUDA_TRY(cudaMalloc(&snap, total));
        auto copy_all = [&](bool save) -> cudaError_t {
          size_t off = 0;
          for (auto& x : st) {
            cudaError_t r = save ? cudaMemcpyAsync(snap + off, x.first, x.second, cudaMemcpyDeviceToDevice, e.stream)
                                 : cudaMemcpyAsync(x.first, snap + off, x.second, cudaMemcpyDeviceToDevice, e.stream);
            if (r != cudaSuccess) return r;
            off += (x.second + 255) & ~size_t(255);
          }
          return cudaSuccess;
        };
        cudaEvent_t a, b;
        float sum = 0.0f;
        cudaError_t r = copy_all(true);
        if (r == cudaSuccess) r = cudaEventCreate(&a);
        if (r == cudaSuccess) r = cudaEventCreate(&b);
        for (uint64_t i = 0; i <= iters && r == cudaSuccess; ++i) {  // launch 0: warm-up
          r = copy_all(false);
          if (r == cudaSuccess) r = flush_l2(e.stream);
          if (r == cudaSuccess) r = cudaEventRecord(a, e.stream);
          if (r == cudaSuccess) launch_select_gen(v, w.nsm, e.stream);
          if (r == cudaSuccess) r = cudaEventRecord(b, e.stream);
          if (r == cudaSuccess) r = cudaEventSynchronize(b);
          float t = 0.0f;
          if (r == cudaSuccess) r = cudaEventElapsedTime(&t, a, b);
          if (i > 0) sum += t;
        }
        if (r == cudaSuccess) r = copy_all(false);
        if (r == cudaSuccess) r = cudaStreamSynchronize(e.stream);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaFree(snap);
        CUDA_TRY(r);
        *ms = (double)sum / (double)(iters ? iters : 1);
        *units = v.Fl;
        return ok();
      }
      default:
        return invalid("mgfwa_time_kernel: unknown kernel");
    }
    // Each timed launch starts from a cold L2: a 256 MB write (> the 126 MB
    // L2) runs before it, outside the events.
    cudaEvent_t a, b;
    CUDA_TRY(cudaEventCreate(&a));
    CUDA_TRY(cudaEventCreate(&b));
    launch();
    double sum = 0.0;
    for (uint64_t i = 0; i < iters; ++i) {
      CUDA_TRY(flush_l2(e.stream));
      CUDA_TRY(cudaEventRecord(a, e.stream));
      launch();
      CUDA_TRY(cudaEventRecord(b, e.stream));
      CUDA_TRY(cudaEventSynchronize(b));
      CUDA_TRY(cudaGetLastError());
      float t = 0.0f;
      CUDA_TRY(cudaEventElapsedTime(&t, a, b));
      sum += t;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *ms = sum / (double)(iters ? iters : 1);
    return ok();
  };
  return fail(ctx, body());
}

int mgfwa_time_fitness(mgfwa_ctx_t ctx, uint64_t iters, double* ms, uint64_t* units) {
  return mgfwa_time_kernel(ctx, MGFWA_KERNEL_FITNESS, iters, ms, units);
}

int mgfwa_validate_config(const mgfwa_config_t* config) {
  if (config == nullptr) return fail(nullptr, invalid("mgfwa_validate_config: null config"));
  return fail(nullptr, validate_config(to_host(config)));
}

int mgfwa_key_hash(const uint64_t* keys, uint64_t n, uint64_t* out) {
  auto body = [&]() -> Status {
    uint64_t *dk = nullptr, *dout = nullptr;
    CUDA_TRY(cudaMalloc(&dk, n * 7 * 8));
    CUDA_TRY(cudaMalloc(&dout, n * 8));
    CUDA_TRY(cudaMemcpy(dk, keys, n * 7 * 8, cudaMemcpyHostToDevice));
    launch_key_hash(dk, n, dout, 0);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpy(out, dout, n * 8, cudaMemcpyDeviceToHost));
    cudaFree(dk);
    cudaFree(dout);
    return ok();
  };
  return fail(nullptr, body());
}

}  // extern "C"
