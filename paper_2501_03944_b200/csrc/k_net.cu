// k_net.cu — the reference's input-space benchmark networks (Nets 1-12,
// SURVEY.md §8(f) rank 2): MlpBlackBox(net_spec(id), weight_seed), the
// candidate is the network input, the output is a scalar
// (/root/reference/proj/src/nets.cpp:36-167).
//
// The weights are fixed and shared by every candidate, so each layer is a
// plain GEMM  Y[rows][out] = act(X[rows][in] . W[out][in]^T + b)  with the
// candidates as rows.  The path is tiny in FLOPs (net 12: 3.65 M MACs per
// candidate) and is evaluated in fp64 with the reference's exact operation
// order — acc = b[o]; acc += w[o][i] * x[i] for ascending i, no FMA
// contraction (nets.cpp:150-160) — so a ReLU network's output is
// bit-identical to the reference's forward() on the same (fp32) input; GELU
// differs only by the device tanh (<= 1-2 ulp per activation).
//
// Layer kernel: 64 x 64 output tile per 256-thread block, 4 x 4 outputs per
// thread, K streamed through shared memory in chunks of 16 (each thread's
// 16 accumulators keep their own ascending-i chain).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <new>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace mgfwa_b200 {

namespace {

constexpr int kT = 64;    // block tile (rows and outputs)
constexpr int kKc = 16;   // K chunk
constexpr int kTh = 256;  // threads per block

struct NetSpecRow {
  int activation;  // 0 relu, 1 gelu
  uint32_t input_dim, hidden_dim, hidden_layers;
};

// net_registry(), nets.cpp:36-55 (output_dim = 1 for every net)
const NetSpecRow kRegistry[12] = {
    {0, 10, 16, 2},     {1, 10, 32, 5},     {0, 20, 16, 5},     {1, 20, 32, 5},
    {0, 100, 64, 8},    {1, 100, 128, 8},   {0, 200, 64, 8},    {1, 200, 128, 8},
    {0, 1000, 256, 11}, {1, 1000, 512, 11}, {0, 2000, 256, 11}, {1, 2000, 512, 11},
};

// gelu, nets.cpp:74-78, same operation order.
__device__ __forceinline__ double gelu_ref(double x) {
  const double k = 0.7978845608028654;
  const double cube = __dmul_rn(__dmul_rn(__dmul_rn(0.044715, x), x), x);
  const double inner = __dmul_rn(k, __dadd_rn(x, cube));
  return __dmul_rn(__dmul_rn(0.5, x), __dadd_rn(1.0, tanh(inner)));
}

struct LayerArgs {
  const float* xf;   // first layer: fp32 candidate rows (stride ldx)
  const double* xd;  // later layers: fp64 activations (stride ldx)
  uint64_t ldx;
  const double* W;   // [out][in]
  const double* b;   // [out]
  double* y;         // [rows][out] (not the last layer)
  float* part;       // last layer: part[row * 2] = output
  uint64_t rows;
  uint32_t in, out;
  int act, last;
  const int* gate;
};

}  // namespace

__global__ void __launch_bounds__(kTh) k_net_layer(LayerArgs a) {
  pdl_enter();
  if (a.gate != nullptr && *a.gate == 0) return;
  __shared__ double sx[kT][kKc + 1];
  __shared__ double sw[kT][kKc + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // out group, row group
  const uint64_t r0 = (uint64_t)blockIdx.x * kT;
  const uint32_t o0 = blockIdx.y * kT;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t o = o0 + tx + 16 * j;
      acc[i][j] = o < a.out ? a.b[o] : 0.0;
    }
  for (uint32_t k0 = 0; k0 < a.in; k0 += kKc) {
    __syncthreads();
    for (int e = threadIdx.x; e < kT * kKc; e += kTh) {
      const int rr = e / kKc, kk = e % kKc;
      const uint64_t r = r0 + rr;
      const uint32_t k = k0 + kk;
      double xv = 0.0;
      if (r < a.rows && k < a.in) xv = a.xf ? (double)a.xf[r * a.ldx + k] : a.xd[r * a.ldx + k];
      sx[rr][kk] = xv;
      const uint32_t o = o0 + rr;
      sw[rr][kk] = (o < a.out && k < a.in) ? a.W[(uint64_t)o * a.in + k] : 0.0;
    }
    __syncthreads();
    const int kn = (int)min((uint32_t)kKc, a.in - k0);
    for (int kk = 0; kk < kn; ++kk) {  // ascending i within each accumulator
      double xv[4], wv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = sx[ty + 16 * i][kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) wv[j] = sw[tx + 16 * j][kk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(wv[j], xv[i]));
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t r = r0 + ty + 16 * i;
    if (r >= a.rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t o = o0 + tx + 16 * j;
      if (o >= a.out) continue;
      double v = acc[i][j];
      if (a.last) {
        a.part[r * 2] = (float)v;
        a.part[r * 2 + 1] = 0.0f;
      } else {
        v = a.act ? gelu_ref(v) : (v > 0.0 ? v : 0.0);  // relu, nets.hpp:48
        a.y[r * a.out + o] = v;
      }
    }
  }
}

struct NetPlan {
  std::vector<LayerArgs> layers;
  double* weights = nullptr;  // all layers' W and b (owned)
  double* act = nullptr;      // two activation buffers [rows][hidden] (owned)
};

bool net_spec_dims(int net_id, uint32_t* input_dim, uint32_t* hidden_dim, uint32_t* layers,
                   int* gelu) {
  if (net_id < 1 || net_id > 12) return false;
  const NetSpecRow& s = kRegistry[net_id - 1];
  if (input_dim) *input_dim = s.input_dim;
  if (hidden_dim) *hidden_dim = s.hidden_dim;
  if (layers) *layers = s.hidden_layers;
  if (gelu) *gelu = s.activation;
  return true;
}

// sampled_layer, nets.cpp:90-108: W[o][i] = U(-1/sqrt(in), 1/sqrt(in)) with
// key (seed, kWeights, layer, 1, o, 0, i); b[o] with key (seed, kWeights,
// layer, 0, o, 0, 0).
static void sample_layer(uint32_t in, uint32_t out, uint64_t layer, uint64_t seed, double* W,
                         double* b) {
  const double bound = 1.0 / std::sqrt((double)in);
  auto uniform = [&](uint64_t it, uint64_t bb, uint64_t n, uint64_t d) {
    const uint64_t h = splitmix64(key_prefix(seed, kWeights, it, bb, n, 0) ^ d);
    const double u = (double)(h >> 11) * 0x1.0p-53;
    return -bound + u * (bound - -bound);
  };
  for (uint32_t o = 0; o < out; ++o) {
    for (uint32_t i = 0; i < in; ++i) W[(uint64_t)o * in + i] = uniform(layer, 1, o, i);
    b[o] = uniform(layer, 0, o, 0);
  }
}

NetPlan* net_plan_create(int net_id, uint64_t weight_seed, const float* X, uint64_t ldx,
                         uint64_t rows, char* err, size_t errlen) {
  uint32_t D, H, L;
  int gelu;
  if (!net_spec_dims(net_id, &D, &H, &L, &gelu)) {
    snprintf(err, errlen, "net id must be in 1..12");
    return nullptr;
  }
  auto* p = new (std::nothrow) NetPlan{};
  if (!p) return nullptr;
  // layer shapes: (D -> H), (L - 1) x (H -> H), (H -> 1)
  std::vector<std::pair<uint32_t, uint32_t>> shapes;
  shapes.push_back({D, H});
  for (uint32_t l = 1; l < L; ++l) shapes.push_back({H, H});
  shapes.push_back({H, 1});
  size_t total = 0;
  for (auto& s : shapes) total += (size_t)s.first * s.second + s.second;
  std::vector<double> host(total);
  size_t off = 0;
  std::vector<size_t> offs;
  for (size_t l = 0; l < shapes.size(); ++l) {
    offs.push_back(off);
    sample_layer(shapes[l].first, shapes[l].second, l, weight_seed, host.data() + off,
                 host.data() + off + (size_t)shapes[l].first * shapes[l].second);
    off += (size_t)shapes[l].first * shapes[l].second + shapes[l].second;
  }
  if (cudaMalloc(&p->weights, total * 8) != cudaSuccess ||
      cudaMemcpy(p->weights, host.data(), total * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMalloc(&p->act, 2 * rows * H * 8) != cudaSuccess) {
    snprintf(err, errlen, "net objective: device allocation failed");
    net_plan_destroy(p);
    return nullptr;
  }
  for (size_t l = 0; l < shapes.size(); ++l) {
    LayerArgs a{};
    a.xf = l == 0 ? X : nullptr;
    a.xd = l == 0 ? nullptr : p->act + ((l - 1) % 2) * rows * H;
    a.ldx = l == 0 ? ldx : H;
    a.W = p->weights + offs[l];
    a.b = a.W + (size_t)shapes[l].first * shapes[l].second;
    a.y = p->act + (l % 2) * rows * H;
    a.rows = rows;
    a.in = shapes[l].first;
    a.out = shapes[l].second;
    a.act = gelu;
    a.last = l + 1 == shapes.size();
    p->layers.push_back(a);
  }
  return p;
}

void net_plan_destroy(NetPlan* p) {
  if (!p) return;
  cudaFree(p->weights);
  cudaFree(p->act);
  delete p;
}

cudaError_t net_fitness_launch(const NetPlan* p, float* part, const int* gate, cudaStream_t s) {
  for (const LayerArgs& l0 : p->layers) {
    LayerArgs a = l0;
    a.part = part;
    a.gate = gate;
    const dim3 grid((unsigned)((a.rows + kT - 1) / kT), (a.out + kT - 1) / kT);
    cudaError_t e = pdl_launch(k_net_layer, grid, kTh, 0, s, a);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace mgfwa_b200
