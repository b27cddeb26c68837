// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" seam over the UNMODIFIED reference engine (compiled from the
// sources under /root/reference/proj by oracle/Makefile into
// oracle/_ref/libmgfwa_ref.so).  It lets the Python test harness and
// bench.py's reference arm call the reference's own run() / operators
// (engine.hpp:71-132, backend.hpp:42-51) on caller-provided arrays.
//
// The objectives the reference does not ship (Rastrigin, Ackley, the
// MLP-weights loss and the LeNet loss) are restated here in
// C++ following the reference conventions (nets.cpp:80-84, 138-167: fp64,
// fixed ascending accumulation) and plugged in through the reference's
// own Objective boundary (backend.hpp:15).  This is the second, independent
// restatement of those objectives; oracle/mgfwa_oracle.c is the first.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "mgfwa/backend.hpp"
#include "mgfwa/config.hpp"
#include "mgfwa/engine.hpp"
#include "mgfwa/nets.hpp"
#include "mgfwa/rng.hpp"

using namespace mgfwa;

extern "C" {

struct ref_config_t {
  uint64_t batches, fireworks, sparks, guides;
  double guide_fraction;
  const double* boosts;
  uint64_t n_boosts;
  double amp_amplify, amp_reduce, initial_amplitude;
  uint64_t max_evaluations;
  double wall_clock_budget_ms;
};

struct ref_objective_desc_t {
  int kind;  // 1 sphere 2 rastrigin 3 ackley 4 mlp-weights 5 lenet 6 net
  uint32_t in_dim, hidden, out_dim, samples;
  uint64_t data_seed;
  int net_id;
  uint64_t weight_seed;
};

struct ref_counters_t {
  uint64_t evaluations_used, iterations, losers_reinitialized,
      nan_evaluations, waves;
};

}  // extern "C"

namespace {

MgfwaConfig to_config(const ref_config_t* c) {
  MgfwaConfig cfg;
  cfg.batches = c->batches;
  cfg.fireworks = c->fireworks;
  cfg.sparks_per_firework = c->sparks;
  cfg.guides_per_firework = c->guides;
  cfg.guide_fraction = c->guide_fraction;
  cfg.boosts.assign(c->boosts, c->boosts + c->n_boosts);
  cfg.amp_amplify = c->amp_amplify;
  cfg.amp_reduce = c->amp_reduce;
  cfg.initial_amplitude = c->initial_amplitude;
  cfg.max_evaluations = c->max_evaluations;
  cfg.wall_clock_budget_ms = c->wall_clock_budget_ms;
  return cfg;
}

SearchSpace to_space(const double* lo, const double* hi, uint64_t d) {
  SearchSpace s;
  s.lower.assign(lo, lo + d);
  s.upper.assign(hi, hi + d);
  return s;
}

EvalBackend to_backend(int workers) {
  return workers <= 0 ? EvalBackend::serial()
                      : EvalBackend::data_parallel(workers);
}

void set_err(char* err, size_t n, const char* msg) {
  if (err && n) {
    std::strncpy(err, msg, n - 1);
    err[n - 1] = 0;
  }
}

constexpr double kPi = 3.14159265358979323846;

// Synthetic dataset, builder-defined; kData = 7 is a new
// stream id beyond rng.hpp:11-18.
struct Dataset {
  uint32_t samples = 0, in_dim = 0, out_dim = 0;
  std::vector<double> X;
  std::vector<int32_t> y;
};

Dataset make_dataset(uint32_t S, uint32_t I, uint32_t O, uint64_t seed) {
  const auto kData = static_cast<RngStream>(7);
  Dataset ds;
  ds.samples = S;
  ds.in_dim = I;
  ds.out_dim = O;
  ds.X.resize(static_cast<size_t>(S) * I);
  ds.y.resize(S);
  std::vector<double> T(static_cast<size_t>(O) * I);
  for (uint32_t o = 0; o < O; ++o)
    for (uint32_t i = 0; i < I; ++i)
      T[static_cast<size_t>(o) * I + i] =
          uniform_sample(RngKey{seed, kData, 1, 0, o, 0, i}, -1.0, 1.0);
  for (uint32_t s = 0; s < S; ++s) {
    for (uint32_t i = 0; i < I; ++i)
      ds.X[static_cast<size_t>(s) * I + i] =
          static_cast<double>(key_hash(RngKey{seed, kData, 0, 0, s, 0, i}) >> 56) /
          256.0;
    int32_t best = 0;
    double best_v = 0.0;
    for (uint32_t o = 0; o < O; ++o) {
      double acc = 0.0;
      for (uint32_t i = 0; i < I; ++i)
        acc += T[static_cast<size_t>(o) * I + i] *
               (ds.X[static_cast<size_t>(s) * I + i] - 0.5);
      if (o == 0 || acc > best_v) {
        best_v = acc;
        best = static_cast<int32_t>(o);
      }
    }
    ds.y[s] = best;
  }
  return ds;
}

double softmax_ce(const double* z, uint32_t n, int32_t label) {
  double m = z[0];
  for (uint32_t o = 1; o < n; ++o) m = std::max(m, z[o]);
  double se = 0.0;
  for (uint32_t o = 0; o < n; ++o) se += std::exp(z[o] - m);
  return (m + std::log(se)) - z[label];
}

struct MlpWeightsLoss {
  std::shared_ptr<const Dataset> ds;
  uint32_t hidden;
  double operator()(std::span<const double> w) const {
    const uint32_t I = ds->in_dim, H = hidden, O = ds->out_dim;
    thread_local std::vector<double> h, z;
    h.assign(H, 0.0);
    z.assign(O, 0.0);
    const double* W1 = w.data();
    const double* b1 = W1 + static_cast<size_t>(H) * I;
    const double* W2 = b1 + H;
    const double* b2 = W2 + static_cast<size_t>(O) * H;
    double total = 0.0;
    for (uint32_t s = 0; s < ds->samples; ++s) {
      const double* x = ds->X.data() + static_cast<size_t>(s) * I;
      for (uint32_t j = 0; j < H; ++j) {
        double acc = b1[j];
        for (uint32_t i = 0; i < I; ++i) acc += W1[static_cast<size_t>(j) * I + i] * x[i];
        h[j] = relu(acc);
      }
      for (uint32_t q = 0; q < O; ++q) {
        double acc = b2[q];
        for (uint32_t j = 0; j < H; ++j) acc += W2[static_cast<size_t>(q) * H + j] * h[j];
        z[q] = acc;
      }
      total += softmax_ce(z.data(), O, ds->y[s]);
    }
    return total / static_cast<double>(ds->samples);
  }
};

// LeNet-5 loss; layer semantics as in oracle/mgfwa_oracle.c f_lenet.
struct LenetLoss {
  std::shared_ptr<const Dataset> ds;
  double operator()(std::span<const double> w) const {
    const double* p = w.data();
    const double* c1w = p; p += 150;
    const double* c1b = p; p += 6;
    const double* c2w = p; p += 2400;
    const double* c2b = p; p += 16;
    const double* f1w = p; p += 48000;
    const double* f1b = p; p += 120;
    const double* f2w = p; p += 10080;
    const double* f2b = p; p += 84;
    const double* f3w = p; p += 840;
    const double* f3b = p;
    thread_local std::vector<double> a1(6 * 28 * 28), p1(6 * 14 * 14),
        a2(16 * 10 * 10), p2(400), h1(120), h2(84), z(10);
    double total = 0.0;
    for (uint32_t s = 0; s < ds->samples; ++s) {
      const double* x = ds->X.data() + static_cast<size_t>(s) * 784;
      for (int c = 0; c < 6; ++c)
        for (int yy = 0; yy < 28; ++yy)
          for (int xx = 0; xx < 28; ++xx) {
            double acc = c1b[c];
            for (int ky = 0; ky < 5; ++ky)
              for (int kx = 0; kx < 5; ++kx) {
                const int iy = yy + ky - 2, ix = xx + kx - 2;
                if (iy < 0 || iy >= 28 || ix < 0 || ix >= 28) continue;
                acc += c1w[c * 25 + ky * 5 + kx] * x[iy * 28 + ix];
              }
            a1[(c * 28 + yy) * 28 + xx] = relu(acc);
          }
      for (int c = 0; c < 6; ++c)
        for (int yy = 0; yy < 14; ++yy)
          for (int xx = 0; xx < 14; ++xx) {
            const double* r0 = &a1[(c * 28 + 2 * yy) * 28 + 2 * xx];
            p1[(c * 14 + yy) * 14 + xx] = 0.25 * (r0[0] + r0[1] + r0[28] + r0[29]);
          }
      for (int c = 0; c < 16; ++c)
        for (int yy = 0; yy < 10; ++yy)
          for (int xx = 0; xx < 10; ++xx) {
            double acc = c2b[c];
            for (int ci = 0; ci < 6; ++ci)
              for (int ky = 0; ky < 5; ++ky)
                for (int kx = 0; kx < 5; ++kx)
                  acc += c2w[((c * 6 + ci) * 5 + ky) * 5 + kx] *
                         p1[(ci * 14 + yy + ky) * 14 + xx + kx];
            a2[(c * 10 + yy) * 10 + xx] = relu(acc);
          }
      for (int c = 0; c < 16; ++c)
        for (int yy = 0; yy < 5; ++yy)
          for (int xx = 0; xx < 5; ++xx) {
            const double* r0 = &a2[(c * 10 + 2 * yy) * 10 + 2 * xx];
            p2[c * 25 + yy * 5 + xx] = 0.25 * (r0[0] + r0[1] + r0[10] + r0[11]);
          }
      for (int j = 0; j < 120; ++j) {
        double acc = f1b[j];
        for (int i = 0; i < 400; ++i) acc += f1w[j * 400 + i] * p2[i];
        h1[j] = relu(acc);
      }
      for (int j = 0; j < 84; ++j) {
        double acc = f2b[j];
        for (int i = 0; i < 120; ++i) acc += f2w[j * 120 + i] * h1[i];
        h2[j] = relu(acc);
      }
      for (int j = 0; j < 10; ++j) {
        double acc = f3b[j];
        for (int i = 0; i < 84; ++i) acc += f3w[j * 84 + i] * h2[i];
        z[j] = acc;
      }
      total += softmax_ce(z.data(), 10, ds->y[s]);
    }
    return total / static_cast<double>(ds->samples);
  }
};

// Holds whatever the Objective closure points at.
struct ObjectiveHolder {
  Objective fn;
  std::shared_ptr<MlpBlackBox> net;
};

ObjectiveHolder make_objective(const ref_objective_desc_t* d) {
  ObjectiveHolder h;
  switch (d->kind) {
    case 1:
      h.fn = Objective(sphere);
      break;
    case 2:
      h.fn = [](std::span<const double> x) {
        double acc = 10.0 * static_cast<double>(x.size());
        for (double v : x) acc += v * v - 10.0 * std::cos(2.0 * kPi * v);
        return acc;
      };
      break;
    case 3:
      h.fn = [](std::span<const double> x) {
        double s2 = 0.0, sc = 0.0;
        for (double v : x) {
          s2 += v * v;
          sc += std::cos(2.0 * kPi * v);
        }
        const double n = static_cast<double>(x.size());
        return -20.0 * std::exp(-0.2 * std::sqrt(s2 / n)) - std::exp(sc / n) +
               20.0 + std::exp(1.0);
      };
      break;
    case 4: {
      auto ds = std::make_shared<const Dataset>(
          make_dataset(d->samples, d->in_dim, d->out_dim, d->data_seed));
      h.fn = MlpWeightsLoss{ds, d->hidden};
      break;
    }
    case 5: {
      auto ds = std::make_shared<const Dataset>(
          make_dataset(d->samples, 784, 10, d->data_seed));
      h.fn = LenetLoss{ds};
      break;
    }
    case 6: {
      h.net = std::make_shared<MlpBlackBox>(net_spec(d->net_id), d->weight_seed);
      auto net = h.net;
      h.fn = [net](std::span<const double> x) { return net->forward(x); };
      break;
    }
    default:
      throw std::invalid_argument("unknown objective kind");
  }
  return h;
}

FireworkState make_state(const double* pos, const double* fit,
                         const double* amp, const double* li, uint64_t B,
                         uint64_t mu, uint64_t D, uint64_t used) {
  FireworkState s{
      BatchCube(B, mu, D, std::vector<double>(pos, pos + B * mu * D)),
      Array2D(B, mu), Array2D(B, mu), Array2D(B, mu), used};
  for (uint64_t i = 0; i < B * mu; ++i) {
    s.fitness.data()[i] = fit ? fit[i] : 0.0;
    s.amplitudes.data()[i] = amp ? amp[i] : 1.0;
    s.last_improvement.data()[i] = li ? li[i] : 0.0;
  }
  return s;
}

}  // namespace

extern "C" {

uint64_t ref_key_hash(uint64_t seed, uint64_t stream, uint64_t iteration,
                      uint64_t b, uint64_t n, uint64_t k, uint64_t d) {
  return key_hash(RngKey{seed, static_cast<RngStream>(stream), iteration, b, n, k, d});
}

int ref_uniform_sample(uint64_t seed, uint64_t stream, uint64_t iteration,
                       uint64_t b, uint64_t n, uint64_t k, uint64_t d,
                       double lo, double hi, double* out) {
  try {
    *out = uniform_sample(
        RngKey{seed, static_cast<RngStream>(stream), iteration, b, n, k, d}, lo, hi);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_config_validate(const ref_config_t* c, char* err, size_t errlen) {
  try {
    to_config(c).validate();
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return -1;
  }
}

uint64_t ref_top_spark_count(const ref_config_t* c) {
  return to_config(c).top_spark_count();
}

double ref_objective_eval(const ref_objective_desc_t* d, const double* x,
                          uint64_t D) {
  auto h = make_objective(d);
  return h.fn(std::span<const double>(x, D));
}

int ref_batched_apply(const ref_objective_desc_t* d, const double* rows,
                      uint64_t B, uint64_t N, uint64_t D, int workers,
                      double* fitness, uint64_t* nan_count) {
  try {
    auto h = make_objective(d);
    EvalStats st;
    BatchCube cube(B, N, D, std::vector<double>(rows, rows + B * N * D));
    Array2D f = batched_apply(h.fn, cube, to_backend(workers), &st);
    std::memcpy(fitness, f.data().data(), sizeof(double) * B * N);
    if (nan_count) *nan_count = st.nan_flagged;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_argmin_per_population(const double* fitness, uint64_t rows,
                              uint64_t cols, uint64_t* index, double* value) {
  Array2D f(rows, cols);
  std::memcpy(f.data().data(), fitness, sizeof(double) * rows * cols);
  const auto best = argmin_per_population(f);
  for (uint64_t b = 0; b < rows; ++b) {
    index[b] = best[b].index;
    value[b] = best[b].value;
  }
  return 0;
}

int ref_initialize(const ref_config_t* c, const double* lower,
                   const double* upper, uint64_t D,
                   const ref_objective_desc_t* d, int workers, uint64_t seed,
                   double* pos, double* fit, double* amp, char* err,
                   size_t errlen) {
  try {
    auto h = make_objective(d);
    auto cfg = to_config(c);
    auto st = initialize(cfg, to_space(lower, upper, D), seed, h.fn,
                         to_backend(workers));
    std::memcpy(pos, st.positions.data().data(), sizeof(double) * st.positions.size());
    std::memcpy(fit, st.fitness.data().data(), sizeof(double) * cfg.batches * cfg.fireworks);
    std::memcpy(amp, st.amplitudes.data().data(), sizeof(double) * cfg.batches * cfg.fireworks);
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return -1;
  }
}

int ref_explode(const double* pos, const double* amp, uint64_t B, uint64_t mu,
                uint64_t D, const ref_config_t* c, uint64_t iteration,
                uint64_t seed, double* sparks) {
  try {
    auto st = make_state(pos, nullptr, amp, nullptr, B, mu, D, 0);
    auto s = explode(st, to_config(c), iteration, seed);
    std::memcpy(sparks, s.positions.data().data(), sizeof(double) * s.positions.size());
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_random_mapping(const double* cand, uint64_t B, uint64_t rows,
                       uint64_t D, uint64_t per, const double* pos,
                       uint64_t mu, const double* lower, const double* upper,
                       uint64_t iteration, uint64_t seed, uint64_t stream,
                       double* out) {
  try {
    auto st = make_state(pos, nullptr, nullptr, nullptr, B, mu, D, 0);
    CandidateSet cs{per, BatchCube(B, rows, D, std::vector<double>(cand, cand + B * rows * D)),
                    Array2D{}};
    auto m = random_mapping(cs, st, to_space(lower, upper, D), iteration, seed,
                            static_cast<RngStream>(stream));
    std::memcpy(out, m.positions.data().data(), sizeof(double) * B * rows * D);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_guiding_vector(const double* sparks, const double* spark_fit,
                       uint64_t B, uint64_t mu, uint64_t D,
                       const ref_config_t* c, double* delta, char* err,
                       size_t errlen) {
  try {
    auto cfg = to_config(c);
    const uint64_t lambda = cfg.sparks_per_firework;
    SparkSet s{lambda, BatchCube(B, mu * lambda, D,
                                 std::vector<double>(sparks, sparks + B * mu * lambda * D)),
               Array2D(B, mu * lambda)};
    std::memcpy(s.fitness.data().data(), spark_fit, sizeof(double) * B * mu * lambda);
    auto dv = guiding_vector(s, cfg);
    std::memcpy(delta, dv.data().data(), sizeof(double) * B * mu * D);
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return -1;
  }
}

int ref_multi_guiding_sparks(const double* pos, const double* delta,
                             uint64_t B, uint64_t mu, uint64_t D,
                             const ref_config_t* c, double* guides) {
  try {
    auto cfg = to_config(c);
    auto st = make_state(pos, nullptr, nullptr, nullptr, B, mu, D, 0);
    BatchCube dv(B, mu, D, std::vector<double>(delta, delta + B * mu * D));
    auto g = multi_guiding_sparks(st, dv, cfg);
    std::memcpy(guides, g.positions.data().data(), sizeof(double) * g.positions.size());
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_select_best(const double* pos, const double* fit, uint64_t B,
                    uint64_t mu, uint64_t D, const double* sparks,
                    const double* spark_fit, uint64_t lambda,
                    const double* guides, const double* guide_fit, uint64_t M,
                    double* new_pos, double* new_fit, double* new_li,
                    double* improved) {
  try {
    auto st = make_state(pos, fit, nullptr, nullptr, B, mu, D, 0);
    SparkSet s{lambda, BatchCube(B, mu * lambda, D,
                                 std::vector<double>(sparks, sparks + B * mu * lambda * D)),
               Array2D(B, mu * lambda)};
    std::memcpy(s.fitness.data().data(), spark_fit, sizeof(double) * B * mu * lambda);
    std::unique_ptr<GuideSet> g;
    if (guides != nullptr && M > 0) {
      g = std::make_unique<GuideSet>(GuideSet{
          M, BatchCube(B, mu * M, D, std::vector<double>(guides, guides + B * mu * M * D)),
          Array2D(B, mu * M)});
      std::memcpy(g->fitness.data().data(), guide_fit, sizeof(double) * B * mu * M);
    }
    auto r = select_best(st, s, g.get());
    std::memcpy(new_pos, r.state.positions.data().data(), sizeof(double) * B * mu * D);
    std::memcpy(new_fit, r.state.fitness.data().data(), sizeof(double) * B * mu);
    std::memcpy(new_li, r.state.last_improvement.data().data(), sizeof(double) * B * mu);
    std::memcpy(improved, r.improved.data().data(), sizeof(double) * B * mu);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_update_amplitudes(const double* amp, const double* improved,
                          uint64_t rows, uint64_t cols, const ref_config_t* c,
                          double max_range, double* out) {
  Array2D a(rows, cols), im(rows, cols);
  std::memcpy(a.data().data(), amp, sizeof(double) * rows * cols);
  std::memcpy(im.data().data(), improved, sizeof(double) * rows * cols);
  auto r = update_amplitudes(a, im, to_config(c), max_range);
  std::memcpy(out, r.data().data(), sizeof(double) * rows * cols);
  return 0;
}

int ref_loser_out(double* pos, double* fit, double* amp, double* li,
                  uint64_t* evaluations_used, uint64_t B, uint64_t mu,
                  uint64_t D, const ref_config_t* c, const double* lower,
                  const double* upper, uint64_t iteration, uint64_t seed,
                  double iterations_remaining, const ref_objective_desc_t* d,
                  int workers, uint64_t* reinit) {
  try {
    auto h = make_objective(d);
    auto st = make_state(pos, fit, amp, li, B, mu, D, *evaluations_used);
    *reinit = loser_out(st, to_config(c), to_space(lower, upper, D), iteration,
                        seed, iterations_remaining, h.fn, to_backend(workers));
    std::memcpy(pos, st.positions.data().data(), sizeof(double) * B * mu * D);
    std::memcpy(fit, st.fitness.data().data(), sizeof(double) * B * mu);
    std::memcpy(amp, st.amplitudes.data().data(), sizeof(double) * B * mu);
    std::memcpy(li, st.last_improvement.data().data(), sizeof(double) * B * mu);
    *evaluations_used = st.evaluations_used;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// run(), engine.cpp:313-423.  Trace arrays are [B][trace_cap].
int ref_run(const ref_config_t* c, const double* lower, const double* upper,
            uint64_t D, const ref_objective_desc_t* d, int workers,
            uint64_t seed, double* best_fitness, double* best_position,
            uint64_t* trace_evals, double* trace_best, double* trace_wall,
            uint64_t trace_cap, ref_counters_t* counters, char* err,
            size_t errlen) {
  try {
    auto h = make_objective(d);
    auto cfg = to_config(c);
    RunRecord rec = run(cfg, to_space(lower, upper, D), h.fn,
                        to_backend(workers), seed);
    const uint64_t B = cfg.batches;
    for (uint64_t b = 0; b < B; ++b) {
      best_fitness[b] = rec.best_fitness[b];
      if (best_position) {
        for (uint64_t j = 0; j < D; ++j)
          best_position[b * D + j] =
              rec.best_position[b].empty() ? 0.0 : rec.best_position[b][j];
      }
      const auto& tr = rec.trace[b];
      for (uint64_t w = 0; w < tr.size() && w < trace_cap; ++w) {
        if (trace_evals) trace_evals[b * trace_cap + w] = tr[w].evaluations;
        if (trace_best) trace_best[b * trace_cap + w] = tr[w].best_fitness;
        if (trace_wall) trace_wall[b * trace_cap + w] = tr[w].wall_ms;
      }
    }
    counters->evaluations_used = rec.evaluations_used;
    counters->iterations = rec.iterations;
    counters->losers_reinitialized = rec.losers_reinitialized;
    counters->nan_evaluations = rec.nan_evaluations;
    counters->waves = rec.trace.empty() ? 0 : rec.trace[0].size();
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return -1;
  }
}

}  // extern "C"
