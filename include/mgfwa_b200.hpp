// mgfwa_b200.hpp — header-only C++ face of the B200 engine, mirroring the
// reference's optimizer interface (/root/reference/proj/include/mgfwa/
// config.hpp, engine.hpp, backend.hpp) over the C-ABI in mgfwa_b200.h.
//
//   mgfwa::b200::MgfwaConfig  == mgfwa::MgfwaConfig      (config.hpp:33-67)
//   mgfwa::b200::SearchSpace  == mgfwa::SearchSpace      (config.hpp:11-28)
//   mgfwa::b200::Objective    replaces the std::function Objective
//                             (backend.hpp:15) with a device descriptor
//   mgfwa::b200::RunRecord    == mgfwa::RunRecord        (engine.hpp:56-67)
//   mgfwa::b200::run(...)     == mgfwa::run(...)         (engine.hpp:130-132)
//
// Errors: MGFWA_EINVAL is rethrown as std::invalid_argument with the
// reference's message; every other failure as std::runtime_error.
#ifndef MGFWA_B200_HPP
#define MGFWA_B200_HPP

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "mgfwa_b200.h"

namespace mgfwa {
namespace b200 {

struct SearchSpace {
  std::vector<double> lower;
  std::vector<double> upper;
  static SearchSpace box(std::size_t dim, double lo, double hi) {
    return SearchSpace{std::vector<double>(dim, lo), std::vector<double>(dim, hi)};
  }
  std::size_t dim() const { return lower.size(); }
};

struct MgfwaConfig {
  std::size_t batches = 8;
  std::size_t fireworks = 5;
  std::size_t sparks_per_firework = 30;
  std::size_t guides_per_firework = 3;
  double guide_fraction = 0.2;
  std::vector<double> boosts = {1.0, 2.0, 4.0};
  double amp_amplify = 1.2;
  double amp_reduce = 0.9;
  double initial_amplitude = 0.0;
  std::uint64_t max_evaluations = 0;
  double wall_clock_budget_ms = 0.0;
};

struct Objective {
  int kind = MGFWA_OBJ_SPHERE;
  std::uint32_t in_dim = 0, hidden = 0, out_dim = 0, samples = 0;
  std::uint64_t data_seed = 0;
  int net_id = 0;
  std::uint64_t weight_seed = 0;
  static Objective sphere() { return Objective{MGFWA_OBJ_SPHERE}; }
  static Objective rastrigin() { return Objective{MGFWA_OBJ_RASTRIGIN}; }
  static Objective ackley() { return Objective{MGFWA_OBJ_ACKLEY}; }
  static Objective mlp_weights(std::uint32_t in = 784, std::uint32_t h = 32, std::uint32_t out = 10,
                               std::uint32_t s = 1024, std::uint64_t seed = 1) {
    return Objective{MGFWA_OBJ_MLP_WEIGHTS, in, h, out, s, seed};
  }
  static Objective lenet(std::uint32_t s = 1024, std::uint64_t seed = 1) {
    return Objective{MGFWA_OBJ_LENET, 784, 0, 10, s, seed};
  }
  // The reference's benchmark network net_id (1..12) with its fixed weights
  // (MlpBlackBox(net_spec(net_id), weight_seed), nets.cpp:36-167).
  static Objective net(int net_id, std::uint64_t weight_seed = 1) {
    Objective o{MGFWA_OBJ_NET};
    o.net_id = net_id;
    o.weight_seed = weight_seed;
    return o;
  }
};

struct TracePoint {
  std::uint64_t evaluations = 0;
  double wall_ms = 0.0;
  double best_fitness = 0.0;
};

struct RunRecord {
  MgfwaConfig config;
  SearchSpace space;
  std::uint64_t seed = 0;
  std::vector<std::vector<TracePoint>> trace;      // [batch][wave]
  std::vector<std::vector<double>> best_position;  // [batch][dim]
  std::vector<double> best_fitness;                // [batch]
  std::uint64_t evaluations_used = 0;
  std::uint64_t iterations = 0;
  std::uint64_t losers_reinitialized = 0;
  std::uint64_t nan_evaluations = 0;
};

namespace detail {
inline void check(int rc, mgfwa_ctx_t ctx = nullptr) {
  if (rc == MGFWA_OK) return;
  const char* m = mgfwa_last_error(ctx);
  const std::string msg = m ? m : "mgfwa_b200 error";
  if (rc == MGFWA_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
inline mgfwa_config_t to_c(const MgfwaConfig& c) {
  return mgfwa_config_t{c.batches,          c.fireworks,   c.sparks_per_firework,
                        c.guides_per_firework, c.guide_fraction, c.boosts.data(),
                        c.boosts.size(),    c.amp_amplify, c.amp_reduce,
                        c.initial_amplitude, c.max_evaluations, c.wall_clock_budget_ms};
}
}  // namespace detail

// One device-resident optimisation context (RAII).
class Engine {
 public:
  Engine(const MgfwaConfig& config, const SearchSpace& space, const Objective& objective,
         std::uint64_t seed, int device = 0)
      : config_(config), space_(space), seed_(seed) {
    if (space.lower.size() != space.upper.size())
      throw std::invalid_argument("SearchSpace: lower/upper must be non-empty and equal length");
    const mgfwa_config_t c = detail::to_c(config);
    const mgfwa_space_t s{space.lower.data(), space.upper.data(), space.lower.size()};
    const mgfwa_objective_t o{objective.kind,    objective.in_dim,    objective.hidden,
                              objective.out_dim, objective.samples,   objective.data_seed,
                              objective.net_id,  objective.weight_seed};
    detail::check(mgfwa_create(&c, &s, &o, seed, device, &ctx_));
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  ~Engine() { mgfwa_destroy(ctx_); }

  void initialize() { detail::check(mgfwa_initialize(ctx_), ctx_); }
  std::uint64_t step(std::uint64_t max_generations) {
    std::uint64_t n = 0;
    detail::check(mgfwa_step(ctx_, max_generations, &n), ctx_);
    return n;
  }

  // run(), engine.cpp:313-423.
  RunRecord run() {
    mgfwa_counters_t cnt{};
    detail::check(mgfwa_run(ctx_, &cnt), ctx_);
    return record();
  }

  RunRecord record() {
    mgfwa_counters_t cnt{};
    detail::check(mgfwa_get_counters(ctx_, &cnt), ctx_);
    const std::size_t B = config_.batches, D = space_.dim();
    RunRecord r;
    r.config = config_;
    r.space = space_;
    r.seed = seed_;
    std::vector<double> bf(B), bp(B * D);
    detail::check(mgfwa_get_best(ctx_, bf.data(), bp.data()), ctx_);
    r.best_fitness = bf;
    r.best_position.resize(B);
    for (std::size_t b = 0; b < B; ++b)
      r.best_position[b].assign(bp.begin() + b * D, bp.begin() + (b + 1) * D);
    std::uint64_t waves = 0;
    detail::check(mgfwa_get_trace(ctx_, nullptr, nullptr, nullptr, 0, &waves), ctx_);
    std::vector<std::uint64_t> te(B * waves);
    std::vector<double> tb(B * waves), tw(B * waves);
    if (waves)
      detail::check(mgfwa_get_trace(ctx_, te.data(), tb.data(), tw.data(), waves, nullptr), ctx_);
    r.trace.assign(B, {});
    for (std::size_t b = 0; b < B; ++b)
      for (std::uint64_t w = 0; w < waves; ++w)
        r.trace[b].push_back({te[b * waves + w], tw[b * waves + w], tb[b * waves + w]});
    r.evaluations_used = cnt.evaluations_used;
    r.iterations = cnt.iterations;
    r.losers_reinitialized = cnt.losers_reinitialized;
    r.nan_evaluations = cnt.nan_evaluations;
    return r;
  }

 private:
  MgfwaConfig config_;
  SearchSpace space_;
  std::uint64_t seed_;
  mgfwa_ctx_t ctx_ = nullptr;
};

// Drop-in for mgfwa::run(config, space, objective, backend, seed).
inline RunRecord run(const MgfwaConfig& config, const SearchSpace& space,
                     const Objective& objective, std::uint64_t seed, int device = 0) {
  Engine e(config, space, objective, seed, device);
  return e.run();
}

}  // namespace b200
}  // namespace mgfwa

#endif  // MGFWA_B200_HPP
