/*
 * mgfwa_oracle.c — TEST INFRASTRUCTURE ONLY (see mgfwa_oracle.h).
 *
 * fp64 CPU restatement of the reference generation path.  Every function
 * names the reference file:line it restates (paths relative to
 * /root/reference/proj).  Compiled with -ffp-contract=off so that the
 * arithmetic order matches the reference build (g++ -O3, no -march: no FMA
 * contraction on baseline x86-64).
 */
#define _POSIX_C_SOURCE 199309L
#include "mgfwa_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ rng */

/* rng.hpp:33-38 */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* rng.hpp:43-52: seed -> stream -> iteration -> b -> n -> k -> d */
uint64_t orc_key_hash(uint64_t seed, uint64_t stream, uint64_t iteration,
                      uint64_t b, uint64_t n, uint64_t k, uint64_t d) {
  uint64_t h = orc_splitmix64(seed);
  h = orc_splitmix64(h ^ stream);
  h = orc_splitmix64(h ^ iteration);
  h = orc_splitmix64(h ^ b);
  h = orc_splitmix64(h ^ n);
  h = orc_splitmix64(h ^ k);
  h = orc_splitmix64(h ^ d);
  return h;
}

/* rng.hpp:55-57 */
double orc_unit_uniform(uint64_t seed, uint64_t stream, uint64_t iteration,
                        uint64_t b, uint64_t n, uint64_t k, uint64_t d) {
  return (double)(orc_key_hash(seed, stream, iteration, b, n, k, d) >> 11) *
         0x1.0p-53;
}

static double uniform_unchecked(uint64_t seed, uint64_t stream,
                                uint64_t iteration, uint64_t b, uint64_t n,
                                uint64_t k, uint64_t d, double lo, double hi) {
  return lo + orc_unit_uniform(seed, stream, iteration, b, n, k, d) * (hi - lo);
}

/* rng.hpp:60-65 */
int orc_uniform_sample(uint64_t seed, uint64_t stream, uint64_t iteration,
                       uint64_t b, uint64_t n, uint64_t k, uint64_t d,
                       double lo, double hi, double* out) {
  if (!(lo <= hi)) return -1;
  *out = uniform_unchecked(seed, stream, iteration, b, n, k, d, lo, hi);
  return 0;
}

/* --------------------------------------------------------------- config */

/* config.cpp:37-40 */
uint64_t orc_top_spark_count(const orc_config_t* c) {
  return (uint64_t)ceil(c->guide_fraction * (double)c->sparks);
}

/* config.cpp:42-79 (same messages, same order) */
const char* orc_config_validate(const orc_config_t* c) {
  if (c->batches == 0 || c->fireworks == 0 || c->sparks == 0)
    return "MgfwaConfig: batches, fireworks and sparks must be positive";
  if (!(c->amp_amplify > 1.0)) return "MgfwaConfig: amp_amplify must be > 1";
  if (!(c->amp_reduce > 0.0 && c->amp_reduce < 1.0))
    return "MgfwaConfig: amp_reduce must be in (0, 1)";
  if (c->max_evaluations == 0 && !(c->wall_clock_budget_ms > 0.0))
    return "MgfwaConfig: at least one budget must be positive";
  if (c->guides > 0) {
    if (!(c->guide_fraction > 0.0 && c->guide_fraction <= 0.5))
      return "MgfwaConfig: guide_fraction must be in (0, 0.5]";
    if (c->guide_fraction * (double)c->sparks < 1.0)
      return "MgfwaConfig: guide_fraction * sparks must be >= 1";
    if (c->sparks < 2 * orc_top_spark_count(c))
      return "MgfwaConfig: sparks must cover disjoint elite and poor sets "
             "(lambda >= 2 * ceil(sigma * lambda))";
    if (c->n_boosts != c->guides)
      return "MgfwaConfig: boosts must list one coefficient per guide";
    if (c->boosts[0] != 1.0)
      return "MgfwaConfig: first boost coefficient must be 1";
    for (uint64_t m = 0; m < c->n_boosts; ++m) {
      if (!(c->boosts[m] > 0.0) || !isfinite(c->boosts[m]))
        return "MgfwaConfig: boost coefficients must be positive finite";
    }
  }
  return NULL;
}

/* config.cpp:25-35 */
const char* orc_space_validate(const double* lower, const double* upper,
                               uint64_t dim) {
  if (dim == 0)
    return "SearchSpace: lower/upper must be non-empty and equal length";
  for (uint64_t d = 0; d < dim; ++d) {
    if (!isfinite(lower[d]) || !isfinite(upper[d]) || !(lower[d] < upper[d]))
      return "SearchSpace: requires lower[d] < upper[d] for all d";
  }
  return NULL;
}

/* config.cpp:17-23 */
double orc_max_range(const double* lower, const double* upper, uint64_t dim) {
  double r = 0.0;
  for (uint64_t d = 0; d < dim; ++d) {
    const double e = upper[d] - lower[d];
    r = r > e ? r : e; /* std::max(range, e) */
  }
  return r;
}

/* ----------------------------------------------------------- objectives */

struct orc_objective {
  int kind;
  uint32_t in_dim, hidden, out_dim, samples;
  uint64_t data_seed;
  uint64_t dim;
  double* X;   /* [samples][in_dim] */
  int32_t* y;  /* [samples] */
};

/*
 * Synthetic dataset (builder decision): 8-bit pixels
 * X[s][i] = (H(seed,kData,0,0,s,0,i) >> 56) / 256 (exact in bf16), labels
 * from a fixed random linear teacher T[o][i] = U(-1,1) on (seed,kData,1,0,o,
 * 0,i): y[s] = argmax_o sum_i T[o][i] * (X[s][i] - 0.5), ascending i, lowest
 * o on ties.
 */
void orc_make_dataset(uint32_t samples, uint32_t in_dim, uint32_t out_dim,
                      uint64_t data_seed, double* X, int32_t* y) {
  double* T = (double*)malloc(sizeof(double) * (size_t)out_dim * in_dim);
  for (uint32_t o = 0; o < out_dim; ++o)
    for (uint32_t i = 0; i < in_dim; ++i)
      T[(size_t)o * in_dim + i] =
          uniform_unchecked(data_seed, ORC_DATA, 1, 0, o, 0, i, -1.0, 1.0);
  for (uint32_t s = 0; s < samples; ++s) {
    for (uint32_t i = 0; i < in_dim; ++i)
      X[(size_t)s * in_dim + i] =
          (double)(orc_key_hash(data_seed, ORC_DATA, 0, 0, s, 0, i) >> 56) /
          256.0;
    int32_t best = 0;
    double best_v = 0.0;
    for (uint32_t o = 0; o < out_dim; ++o) {
      double acc = 0.0;
      for (uint32_t i = 0; i < in_dim; ++i)
        acc += T[(size_t)o * in_dim + i] * (X[(size_t)s * in_dim + i] - 0.5);
      if (o == 0 || acc > best_v) {
        best_v = acc;
        best = (int32_t)o;
      }
    }
    y[s] = best;
  }
  free(T);
}

static uint64_t lenet_dim(void) {
  /* conv1 6x1x5x5+6, conv2 16x6x5x5+16, fc 400->120->84->10 */
  return (6 * 25 + 6) + (16 * 6 * 25 + 16) + (400 * 120 + 120) +
         (120 * 84 + 84) + (84 * 10 + 10);
}

orc_objective_t* orc_objective_create(int kind, uint32_t in_dim,
                                      uint32_t hidden, uint32_t out_dim,
                                      uint32_t samples, uint64_t data_seed) {
  orc_objective_t* o = (orc_objective_t*)calloc(1, sizeof(orc_objective_t));
  o->kind = kind;
  o->in_dim = in_dim;
  o->hidden = hidden;
  o->out_dim = out_dim;
  o->samples = samples;
  o->data_seed = data_seed;
  if (kind == ORC_OBJ_MLP_WEIGHTS) {
    o->dim = (uint64_t)hidden * in_dim + hidden + (uint64_t)out_dim * hidden +
             out_dim;
  } else if (kind == ORC_OBJ_LENET) {
    o->in_dim = in_dim = 784;
    o->out_dim = out_dim = 10;
    o->dim = lenet_dim();
  } else {
    o->dim = 0; /* analytic: any dimension */
  }
  if (kind == ORC_OBJ_MLP_WEIGHTS || kind == ORC_OBJ_LENET) {
    o->X = (double*)malloc(sizeof(double) * (size_t)samples * in_dim);
    o->y = (int32_t*)malloc(sizeof(int32_t) * samples);
    orc_make_dataset(samples, in_dim, out_dim, data_seed, o->X, o->y);
  }
  return o;
}

void orc_objective_destroy(orc_objective_t* o) {
  if (!o) return;
  free(o->X);
  free(o->y);
  free(o);
}

uint64_t orc_objective_dim(const orc_objective_t* o) { return o->dim; }
const double* orc_objective_data(const orc_objective_t* o) { return o->X; }
const int32_t* orc_objective_labels(const orc_objective_t* o) { return o->y; }

/* sphere, nets.cpp:80-84: fixed ascending order */
static double f_sphere(const double* x, uint64_t n) {
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i) acc += x[i] * x[i];
  return acc;
}

static const double kPi = 3.14159265358979323846;

/* Rastrigin (builder-defined, unshifted): 10 D + sum(x^2 - 10 cos 2 pi x) */
static double f_rastrigin(const double* x, uint64_t n) {
  double acc = 10.0 * (double)n;
  for (uint64_t i = 0; i < n; ++i)
    acc += x[i] * x[i] - 10.0 * cos(2.0 * kPi * x[i]);
  return acc;
}

/* Ackley (builder-defined, unshifted) */
static double f_ackley(const double* x, uint64_t n) {
  double s2 = 0.0, sc = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    s2 += x[i] * x[i];
    sc += cos(2.0 * kPi * x[i]);
  }
  const double dn = (double)n;
  return -20.0 * exp(-0.2 * sqrt(s2 / dn)) - exp(sc / dn) + 20.0 + exp(1.0);
}

/* log-softmax cross-entropy of one logit row */
static double cross_entropy(const double* z, uint32_t nout, int32_t label) {
  double m = z[0];
  for (uint32_t o = 1; o < nout; ++o) m = z[o] > m ? z[o] : m;
  double se = 0.0;
  for (uint32_t o = 0; o < nout; ++o) se += exp(z[o] - m);
  return (m + log(se)) - z[label];
}

/*
 * MLP-weights loss (new objective; pattern nets.cpp:138-167).  The candidate
 * w parameterises W1[H][I], b1[H], W2[O][H], b2[O] in the reference Layer
 * order (weights row-major then bias, nets.hpp:60-65).  Each unit starts
 * from its bias and accumulates in ascending input order; ReLU on the
 * hidden layer only.  f(w) = mean_s CE(softmax(z_s), y_s).
 */
static double f_mlp_weights(const orc_objective_t* o, const double* w) {
  const uint32_t I = o->in_dim, H = o->hidden, O = o->out_dim;
  const double* W1 = w;
  const double* b1 = W1 + (size_t)H * I;
  const double* W2 = b1 + H;
  const double* b2 = W2 + (size_t)O * H;
  double* h = (double*)malloc(sizeof(double) * H);
  double* z = (double*)malloc(sizeof(double) * O);
  double total = 0.0;
  for (uint32_t s = 0; s < o->samples; ++s) {
    const double* x = o->X + (size_t)s * I;
    for (uint32_t j = 0; j < H; ++j) {
      double acc = b1[j];
      const double* wr = W1 + (size_t)j * I;
      for (uint32_t i = 0; i < I; ++i) acc += wr[i] * x[i];
      h[j] = acc > 0.0 ? acc : 0.0;
    }
    for (uint32_t q = 0; q < O; ++q) {
      double acc = b2[q];
      const double* wr = W2 + (size_t)q * H;
      for (uint32_t j = 0; j < H; ++j) acc += wr[j] * h[j];
      z[q] = acc;
    }
    total += cross_entropy(z, O, o->y[s]);
  }
  free(h);
  free(z);
  return total / (double)o->samples;
}

/*
 * LeNet-5 loss (new objective, builder-defined):
 * conv5x5 1->6 pad 2 (28x28) -> ReLU -> 2x2 avg-pool (14x14)
 * -> conv5x5 6->16 valid (10x10) -> ReLU -> 2x2 avg-pool (5x5)
 * -> fc 400->120 -> ReLU -> fc 120->84 -> ReLU -> fc 84->10 -> CE.
 * Parameter order: conv1 W[6][1][5][5], b[6]; conv2 W[16][6][5][5], b[16];
 * fc1 W[120][400], b; fc2 W[84][120], b; fc3 W[10][84], b.  Flatten order
 * of the 16x5x5 map is c-major (c, y, x).
 */
static double f_lenet(const orc_objective_t* o, const double* w) {
  const double* c1w = w;
  const double* c1b = c1w + 150;
  const double* c2w = c1b + 6;
  const double* c2b = c2w + 2400;
  const double* f1w = c2b + 16;
  const double* f1b = f1w + 48000;
  const double* f2w = f1b + 120;
  const double* f2b = f2w + 10080;
  const double* f3w = f2b + 84;
  const double* f3b = f3w + 840;
  double a1[6][28][28], p1[6][14][14], a2[16][10][10], p2[400];
  double h1[120], h2[84], z[10];
  double total = 0.0;
  for (uint32_t s = 0; s < o->samples; ++s) {
    const double* x = o->X + (size_t)s * 784;
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
          a1[c][yy][xx] = acc > 0.0 ? acc : 0.0;
        }
    for (int c = 0; c < 6; ++c)
      for (int yy = 0; yy < 14; ++yy)
        for (int xx = 0; xx < 14; ++xx)
          p1[c][yy][xx] = 0.25 * (a1[c][2 * yy][2 * xx] + a1[c][2 * yy][2 * xx + 1] +
                                  a1[c][2 * yy + 1][2 * xx] +
                                  a1[c][2 * yy + 1][2 * xx + 1]);
    for (int c = 0; c < 16; ++c)
      for (int yy = 0; yy < 10; ++yy)
        for (int xx = 0; xx < 10; ++xx) {
          double acc = c2b[c];
          for (int ci = 0; ci < 6; ++ci)
            for (int ky = 0; ky < 5; ++ky)
              for (int kx = 0; kx < 5; ++kx)
                acc += c2w[((c * 6 + ci) * 5 + ky) * 5 + kx] *
                       p1[ci][yy + ky][xx + kx];
          a2[c][yy][xx] = acc > 0.0 ? acc : 0.0;
        }
    for (int c = 0; c < 16; ++c)
      for (int yy = 0; yy < 5; ++yy)
        for (int xx = 0; xx < 5; ++xx)
          p2[c * 25 + yy * 5 + xx] =
              0.25 * (a2[c][2 * yy][2 * xx] + a2[c][2 * yy][2 * xx + 1] +
                      a2[c][2 * yy + 1][2 * xx] + a2[c][2 * yy + 1][2 * xx + 1]);
    for (int j = 0; j < 120; ++j) {
      double acc = f1b[j];
      for (int i = 0; i < 400; ++i) acc += f1w[j * 400 + i] * p2[i];
      h1[j] = acc > 0.0 ? acc : 0.0;
    }
    for (int j = 0; j < 84; ++j) {
      double acc = f2b[j];
      for (int i = 0; i < 120; ++i) acc += f2w[j * 120 + i] * h1[i];
      h2[j] = acc > 0.0 ? acc : 0.0;
    }
    for (int j = 0; j < 10; ++j) {
      double acc = f3b[j];
      for (int i = 0; i < 84; ++i) acc += f3w[j * 84 + i] * h2[i];
      z[j] = acc;
    }
    total += cross_entropy(z, 10, o->y[s]);
  }
  return total / (double)o->samples;
}

double orc_objective_eval(const orc_objective_t* o, const double* x,
                          uint64_t dim) {
  switch (o->kind) {
    case ORC_OBJ_SPHERE: return f_sphere(x, dim);
    case ORC_OBJ_RASTRIGIN: return f_rastrigin(x, dim);
    case ORC_OBJ_ACKLEY: return f_ackley(x, dim);
    case ORC_OBJ_MLP_WEIGHTS: return f_mlp_weights(o, x);
    case ORC_OBJ_LENET: return f_lenet(o, x);
    default: return NAN;
  }
}

/* backend.cpp:15-24 + 28-67 (serial order; result is order-independent) */
uint64_t orc_batched_apply(const orc_objective_t* obj, const double* rows,
                           uint64_t nrows, uint64_t dim, double* fitness) {
  uint64_t nan_count = 0;
  for (uint64_t r = 0; r < nrows; ++r) {
    const double v = orc_objective_eval(obj, rows + r * dim, dim);
    if (isnan(v)) {
      ++nan_count;
      fitness[r] = INFINITY;
    } else {
      fitness[r] = v;
    }
  }
  return nan_count;
}

/* backend.cpp:69-83: strict <, lowest index on ties, all-inf -> 0 */
void orc_argmin_per_population(const double* fitness, uint64_t rows,
                               uint64_t cols, uint64_t* index,
                               double* value) {
  for (uint64_t b = 0; b < rows; ++b) {
    uint64_t arg = 0;
    double val = fitness[b * cols];
    for (uint64_t n = 1; n < cols; ++n) {
      if (fitness[b * cols + n] < val) {
        val = fitness[b * cols + n];
        arg = n;
      }
    }
    index[b] = arg;
    value[b] = val;
  }
}

/* --------------------------------------------------------------- engine */

/* engine.cpp:22-41 (std::min / std::max semantics: keep first on ties) */
void orc_population_range(const double* pos, uint64_t B, uint64_t mu,
                          uint64_t D, double* lo, double* hi) {
  for (uint64_t b = 0; b < B; ++b)
    for (uint64_t d = 0; d < D; ++d) {
      double mn = pos[(b * mu) * D + d];
      double mx = mn;
      for (uint64_t n = 1; n < mu; ++n) {
        const double v = pos[(b * mu + n) * D + d];
        mn = (v < mn) ? v : mn; /* std::min(mn, v) */
        mx = (mx < v) ? v : mx; /* std::max(mx, v) */
      }
      lo[b * D + d] = mn;
      hi[b * D + d] = mx;
    }
}

/* engine.cpp:45-64 */
void orc_initialize_positions(const orc_config_t* c, const double* lower,
                              const double* upper, uint64_t D, uint64_t seed,
                              double* pos) {
  uint64_t idx = 0;
  for (uint64_t b = 0; b < c->batches; ++b)
    for (uint64_t n = 0; n < c->fireworks; ++n)
      for (uint64_t d = 0; d < D; ++d)
        pos[idx++] = uniform_unchecked(seed, ORC_INIT, 0, b, n, 0, d, lower[d],
                                       upper[d]);
}

/* engine.cpp:78-101 */
void orc_explode(const double* pos, const double* amp, uint64_t B,
                 uint64_t mu, uint64_t D, uint64_t lambda, uint64_t iteration,
                 uint64_t seed, double* sparks) {
  uint64_t idx = 0;
  for (uint64_t b = 0; b < B; ++b)
    for (uint64_t n = 0; n < mu; ++n) {
      const double a = amp[b * mu + n];
      for (uint64_t k = 0; k < lambda; ++k)
        for (uint64_t d = 0; d < D; ++d) {
          const double u = uniform_unchecked(seed, ORC_EXPLODE, iteration, b, n,
                                             k, d, -1.0, 1.0);
          sparks[idx++] = pos[(b * mu + n) * D + d] + u * a;
        }
    }
}

/* engine.cpp:103-131; SearchSpace::contains is inclusive (config.hpp:22) */
void orc_random_mapping(double* cand, uint64_t B, uint64_t rows, uint64_t D,
                        uint64_t per, const double* pos, uint64_t mu,
                        const double* lower, const double* upper,
                        uint64_t iteration, uint64_t seed, uint64_t stream) {
  double* lo = (double*)malloc(sizeof(double) * B * D);
  double* hi = (double*)malloc(sizeof(double) * B * D);
  orc_population_range(pos, B, mu, D, lo, hi);
  uint64_t idx = 0;
  for (uint64_t b = 0; b < B; ++b)
    for (uint64_t r = 0; r < rows; ++r) {
      const uint64_t n = r / per, k = r % per;
      for (uint64_t d = 0; d < D; ++d, ++idx) {
        const double x = cand[idx];
        if (!(x >= lower[d] && x <= upper[d])) {
          cand[idx] = uniform_unchecked(seed, stream, iteration, b, n, k, d,
                                        lo[b * D + d], hi[b * D + d]);
        }
      }
    }
  free(lo);
  free(hi);
}

typedef struct {
  double f;
  uint64_t i;
} rank_item;

static int rank_cmp(const void* a, const void* b) {
  const rank_item* x = (const rank_item*)a;
  const rank_item* y = (const rank_item*)b;
  /* engine.cpp:152-157: (fitness asc, index asc); a total order. */
  if (x->f != y->f) return x->f < y->f ? -1 : 1;
  return x->i < y->i ? -1 : (x->i > y->i ? 1 : 0);
}

/* engine.cpp:133-172 */
int orc_guiding_vector(const double* sparks, const double* spark_fit,
                       uint64_t B, uint64_t mu, uint64_t lambda, uint64_t D,
                       uint64_t top, double* delta) {
  if (lambda < 2 * top) return -1;
  rank_item* order = (rank_item*)malloc(sizeof(rank_item) * lambda);
  for (uint64_t b = 0; b < B; ++b)
    for (uint64_t n = 0; n < mu; ++n) {
      for (uint64_t k = 0; k < lambda; ++k) {
        order[k].f = spark_fit[(b * mu + n) * lambda + k];
        order[k].i = k;
      }
      qsort(order, lambda, sizeof(rank_item), rank_cmp);
      double* out = delta + (b * mu + n) * D;
      for (uint64_t d = 0; d < D; ++d) out[d] = 0.0;
      for (uint64_t t = 0; t < top; ++t) {
        const double* best = sparks + ((b * mu + n) * lambda + order[t].i) * D;
        const double* worst =
            sparks + ((b * mu + n) * lambda + order[lambda - top + t].i) * D;
        for (uint64_t d = 0; d < D; ++d) out[d] += best[d] - worst[d];
      }
      for (uint64_t d = 0; d < D; ++d) out[d] /= (double)top;
    }
  free(order);
  return 0;
}

/* engine.cpp:174-196 */
void orc_multi_guiding_sparks(const double* pos, const double* delta,
                              uint64_t B, uint64_t mu, uint64_t D,
                              const double* boosts, uint64_t M,
                              double* guides) {
  uint64_t idx = 0;
  for (uint64_t b = 0; b < B; ++b)
    for (uint64_t n = 0; n < mu; ++n)
      for (uint64_t m = 0; m < M; ++m)
        for (uint64_t d = 0; d < D; ++d)
          guides[idx++] = pos[(b * mu + n) * D + d] +
                          boosts[m] * delta[(b * mu + n) * D + d];
}

/* engine.cpp:198-242: firework, then sparks k up, then guides m up, strict < */
void orc_select_best(const double* pos, const double* fit, uint64_t B,
                     uint64_t mu, uint64_t D, const double* sparks,
                     const double* spark_fit, uint64_t lambda,
                     const double* guides, const double* guide_fit,
                     uint64_t M, double* new_pos, double* new_fit,
                     double* new_li, double* improved) {
  for (uint64_t b = 0; b < B; ++b)
    for (uint64_t n = 0; n < mu; ++n) {
      const uint64_t f = b * mu + n;
      double best_fit = fit[f];
      const double* best_row = pos + f * D;
      for (uint64_t k = 0; k < lambda; ++k) {
        if (spark_fit[f * lambda + k] < best_fit) {
          best_fit = spark_fit[f * lambda + k];
          best_row = sparks + (f * lambda + k) * D;
        }
      }
      if (guides != NULL) {
        for (uint64_t m = 0; m < M; ++m) {
          if (guide_fit[f * M + m] < best_fit) {
            best_fit = guide_fit[f * M + m];
            best_row = guides + (f * M + m) * D;
          }
        }
      }
      memmove(new_pos + f * D, best_row, sizeof(double) * D);
      const double old = fit[f];
      new_fit[f] = best_fit;
      const double gain = old - best_fit;
      new_li[f] = (0.0 < gain) ? gain : 0.0; /* std::max(0.0, old - best) */
      improved[f] = best_fit < old ? 1.0 : 0.0;
    }
}

/* engine.cpp:244-256 (std::clamp(v, lo, hi)) */
void orc_update_amplitudes(const double* amp, const double* improved,
                           uint64_t n, double amp_amplify, double amp_reduce,
                           double max_range, double* out) {
  const double lo = 1e-12 * max_range;
  for (uint64_t i = 0; i < n; ++i) {
    const double factor = improved[i] != 0.0 ? amp_amplify : amp_reduce;
    const double v = amp[i] * factor;
    out[i] = v < lo ? lo : (max_range < v ? max_range : v);
  }
}

/* engine.cpp:258-311 */
uint64_t orc_loser_out(double* pos, double* fit, double* amp, double* li,
                       uint64_t B, uint64_t mu, uint64_t D,
                       const orc_config_t* c, const double* lower,
                       const double* upper, uint64_t iteration, uint64_t seed,
                       double iterations_remaining, const orc_objective_t* obj,
                       uint64_t* nan_count) {
  if (!(iterations_remaining > 0.0)) return 0;
  uint64_t* bi = (uint64_t*)malloc(sizeof(uint64_t) * B);
  double* bv = (double*)malloc(sizeof(double) * B);
  orc_argmin_per_population(fit, B, mu, bi, bv);
  uint64_t* losers = (uint64_t*)malloc(sizeof(uint64_t) * B * mu);
  uint64_t nl = 0;
  for (uint64_t b = 0; b < B; ++b)
    for (uint64_t n = 0; n < mu; ++n) {
      if (n == bi[b]) continue;
      const double projected =
          fit[b * mu + n] - li[b * mu + n] * iterations_remaining;
      if (projected > bv[b]) losers[nl++] = b * mu + n;
    }
  if (nl > 0) {
    const double fresh_amp =
        c->initial_amplitude > 0.0 ? c->initial_amplitude
                                   : 0.5 * orc_max_range(lower, upper, D);
    double* fresh = (double*)malloc(sizeof(double) * nl * D);
    double* ffit = (double*)malloc(sizeof(double) * nl);
    for (uint64_t i = 0; i < nl; ++i) {
      const uint64_t b = losers[i] / mu, n = losers[i] % mu;
      for (uint64_t d = 0; d < D; ++d)
        fresh[i * D + d] = uniform_unchecked(seed, ORC_REINIT, iteration, b, n,
                                             0, d, lower[d], upper[d]);
    }
    *nan_count += orc_batched_apply(obj, fresh, nl, D, ffit);
    for (uint64_t i = 0; i < nl; ++i) {
      const uint64_t f = losers[i];
      memcpy(pos + f * D, fresh + i * D, sizeof(double) * D);
      fit[f] = ffit[i];
      amp[f] = fresh_amp;
      li[f] = 0.0;
    }
    free(fresh);
    free(ffit);
  }
  free(bi);
  free(bv);
  free(losers);
  return nl;
}

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec * 1e3 + (double)ts.tv_nsec * 1e-6;
}

/* engine.cpp:313-423 */
const char* orc_run(const orc_config_t* c, const double* lower,
                    const double* upper, uint64_t D,
                    const orc_objective_t* obj, uint64_t seed,
                    double* best_fitness, double* best_position,
                    uint64_t* trace_evals, double* trace_best,
                    double* trace_wall_ms, uint64_t trace_cap,
                    orc_counters_t* counters) {
  const char* err = orc_config_validate(c);
  if (err) return err;
  err = orc_space_validate(lower, upper, D);
  if (err) return err;
  const uint64_t B = c->batches, mu = c->fireworks, lambda = c->sparks,
                 M = c->guides;
  if (c->max_evaluations > 0 && c->max_evaluations < B * mu)
    return "budget too small: needs at least B * mu evaluations";

  const double start = now_ms();
  uint64_t nan_count = 0;
  const double max_range = orc_max_range(lower, upper, D);
  const double a0 =
      c->initial_amplitude > 0.0 ? c->initial_amplitude : 0.5 * max_range;

  double* pos = (double*)malloc(sizeof(double) * B * mu * D);
  double* fit = (double*)malloc(sizeof(double) * B * mu);
  double* amp = (double*)malloc(sizeof(double) * B * mu);
  double* li = (double*)calloc(B * mu, sizeof(double));
  orc_initialize_positions(c, lower, upper, D, seed, pos);
  nan_count += orc_batched_apply(obj, pos, B * mu, D, fit);
  for (uint64_t i = 0; i < B * mu; ++i) amp[i] = a0;
  uint64_t used = B * mu;

  double* sparks = (double*)malloc(sizeof(double) * B * mu * lambda * D);
  double* sfit = (double*)malloc(sizeof(double) * B * mu * lambda);
  double* guides = M ? (double*)malloc(sizeof(double) * B * mu * M * D) : NULL;
  double* gfit = M ? (double*)malloc(sizeof(double) * B * mu * M) : NULL;
  double* delta = (double*)malloc(sizeof(double) * B * mu * D);
  double* npos = (double*)malloc(sizeof(double) * B * mu * D);
  double* nfit = (double*)malloc(sizeof(double) * B * mu);
  double* nli = (double*)malloc(sizeof(double) * B * mu);
  double* improved = (double*)malloc(sizeof(double) * B * mu);
  uint64_t* bi = (uint64_t*)malloc(sizeof(uint64_t) * B);
  double* bv = (double*)malloc(sizeof(double) * B);
  const uint64_t top = orc_top_spark_count(c);
  const uint64_t wave = B * mu * (lambda + M);

  for (uint64_t b = 0; b < B; ++b) best_fitness[b] = INFINITY;
  uint64_t waves = 0, iteration = 0, losers_total = 0;

#define RECORD_WAVE(wall)                                                   \
  do {                                                                      \
    orc_argmin_per_population(fit, B, mu, bi, bv);                          \
    for (uint64_t b = 0; b < B; ++b) {                                      \
      if (bv[b] < best_fitness[b]) {                                        \
        best_fitness[b] = bv[b];                                            \
        memcpy(best_position + b * D, pos + (b * mu + bi[b]) * D,           \
               sizeof(double) * D);                                         \
      }                                                                     \
      if (waves < trace_cap) {                                              \
        trace_evals[b * trace_cap + waves] = used;                          \
        trace_best[b * trace_cap + waves] = best_fitness[b];                \
        if (trace_wall_ms) trace_wall_ms[b * trace_cap + waves] = (wall);   \
      }                                                                     \
    }                                                                       \
    ++waves;                                                                \
  } while (0)

  RECORD_WAVE(now_ms() - start);
  const double init_ms = now_ms() - start;

  for (;;) {
    if (c->max_evaluations > 0 && used >= c->max_evaluations) break;
    if (c->wall_clock_budget_ms > 0.0 &&
        now_ms() - start >= c->wall_clock_budget_ms)
      break;
    ++iteration;
    orc_explode(pos, amp, B, mu, D, lambda, iteration, seed, sparks);
    orc_random_mapping(sparks, B, mu * lambda, D, lambda, pos, mu, lower,
                       upper, iteration, seed, ORC_MAPPING);
    nan_count += orc_batched_apply(obj, sparks, B * mu * lambda, D, sfit);
    if (M == 0) {
      orc_select_best(pos, fit, B, mu, D, sparks, sfit, lambda, NULL, NULL, 0,
                      npos, nfit, nli, improved);
    } else {
      orc_guiding_vector(sparks, sfit, B, mu, lambda, D, top, delta);
      orc_multi_guiding_sparks(pos, delta, B, mu, D, c->boosts, M, guides);
      orc_random_mapping(guides, B, mu * M, D, M, pos, mu, lower, upper,
                         iteration, seed, ORC_GUIDE);
      nan_count += orc_batched_apply(obj, guides, B * mu * M, D, gfit);
      orc_select_best(pos, fit, B, mu, D, sparks, sfit, lambda, guides, gfit,
                      M, npos, nfit, nli, improved);
    }
    used += wave;
    memcpy(pos, npos, sizeof(double) * B * mu * D);
    memcpy(fit, nfit, sizeof(double) * B * mu);
    memcpy(li, nli, sizeof(double) * B * mu);
    orc_update_amplitudes(amp, improved, B * mu, c->amp_amplify,
                          c->amp_reduce, max_range, amp);

    double iters_rem = 0.0;
    if (c->max_evaluations > 0) {
      const uint64_t left =
          c->max_evaluations > used ? c->max_evaluations - used : 0;
      iters_rem = (double)left / (double)wave;
    } else {
      const double t = now_ms() - start;
      const double avg = (t - init_ms) / (double)iteration;
      if (avg > 0.0) {
        const double rem = c->wall_clock_budget_ms - t;
        iters_rem = (rem > 0.0 ? rem : 0.0) / avg;
      }
    }
    const uint64_t nl = orc_loser_out(pos, fit, amp, li, B, mu, D, c, lower,
                                      upper, iteration, seed, iters_rem, obj,
                                      &nan_count);
    used += nl;
    losers_total += nl;
    RECORD_WAVE(now_ms() - start);
  }
#undef RECORD_WAVE

  counters->evaluations_used = used;
  counters->iterations = iteration;
  counters->losers_reinitialized = losers_total;
  counters->nan_evaluations = nan_count;
  counters->waves = waves;
  free(pos); free(fit); free(amp); free(li); free(sparks); free(sfit);
  free(guides); free(gfit); free(delta); free(npos); free(nfit); free(nli);
  free(improved); free(bi); free(bv);
  return NULL;
}
