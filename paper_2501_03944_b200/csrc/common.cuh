// common.cuh — shared device helpers for the B200 MGFWA engine (sm_100a).
//
// Counter-based RNG (bit-exact restatement of rng.hpp:33-65), fp64 draw
// arithmetic without FMA contraction (so that spark/guide/mapping values are
// the correctly-rounded fp32 image of the reference's fp64 values on equal
// inputs), warp reductions, error helpers.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

namespace mgfwa_b200 {

// RngStream, rng.hpp:11-18, plus kData (builder-defined synthetic data).
enum : uint64_t {
  kInit = 1,
  kExplode = 2,
  kMapping = 3,
  kGuide = 4,
  kReinit = 5,
  kWeights = 6,
  kData = 7
};

// Objective kinds (include/mgfwa_b200.h MGFWA_OBJ_*).
enum : int {
  OBJ_SPHERE = 1,
  OBJ_RASTRIGIN = 2,
  OBJ_ACKLEY = 3,
  OBJ_MLP_WEIGHTS = 4,
  OBJ_LENET = 5
};

// rng.hpp:33-38
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// rng.hpp:43-52 absorbed up to and including field k; the per-coordinate
// hash is then splitmix64(prefix ^ d) — one mixer round per draw.
__host__ __device__ __forceinline__ uint64_t key_prefix(uint64_t seed,
                                                        uint64_t stream,
                                                        uint64_t it, uint64_t b,
                                                        uint64_t n,
                                                        uint64_t k) {
  uint64_t h = splitmix64(seed);
  h = splitmix64(h ^ stream);
  h = splitmix64(h ^ it);
  h = splitmix64(h ^ b);
  h = splitmix64(h ^ n);
  return splitmix64(h ^ k);
}

// ---- per-coordinate draws with the key prefix hoisted (the explode hot loop)
// splitmix64(pre ^ d) (rng.hpp:33-38) for d < 2^32, restated for 32-bit ALUs:
//  * the mixer's "+ gamma" and the prefix's high word fold into one 64-bit
//    addend, so (pre ^ d) + gamma = (pre_lo ^ d) + addend is one IMAD.WIDE
//    (FMA pipe) instead of a carry-chained IADD3 pair (ALU pipe);
//  * the final "z ^ (z >> 31)" is not materialised: the draw only needs bits
//    11..63 of it, and (z ^ (z >> 31)) >> 11 = (z >> 11) ^ (z >> 42).
// MixState holds z before that final xorshift; the unit_*_z helpers below
// produce exactly unit_d1 / unit_pm1 / unit_u53 of splitmix64(pre ^ d).
struct DrawKey {
  uint32_t lo;      // low word of the prefix
  uint64_t addend;  // ((pre_hi + gamma_hi) << 32) | gamma_lo
};
__host__ __device__ __forceinline__ DrawKey draw_key(uint64_t pre) {
  const uint64_t g = 0x9E3779B97F4A7C15ull;
  const uint32_t hi = (uint32_t)(pre >> 32) + (uint32_t)(g >> 32);
  return DrawKey{(uint32_t)pre, ((uint64_t)hi << 32) | (g & 0xFFFFFFFFull)};
}
struct MixState {
  uint32_t lo, hi;
};
#ifndef MIX_MUL_PTX
#define MIX_MUL_PTX 1  // 64-bit multiply as 1 wide + 2 accumulating IMADs (C4 explode 93.1 -> 90.5 us, C2 equal)
#endif
#ifdef __CUDA_ARCH__
// x * C mod 2^64 as one wide and two accumulating 32-bit multiply-adds
__device__ __forceinline__ uint64_t mul64_const(uint64_t x, uint32_t clo, uint32_t chi) {
  uint64_t r;
  asm("{\n\t.reg .u32 xl, xh, rl, rh;\n\t"
      "mov.b64 {xl, xh}, %1;\n\t"
      "mul.wide.u32 %0, xl, %2;\n\t"
      "mov.b64 {rl, rh}, %0;\n\t"
      "mad.lo.u32 rh, xl, %3, rh;\n\t"
      "mad.lo.u32 rh, xh, %2, rh;\n\t"
      "mov.b64 %0, {rl, rh};\n\t}"
      : "=l"(r)
      : "l"(x), "r"(clo), "r"(chi));
  return r;
}
#endif
// `one` must be 1 at run time but opaque to the compiler (so the multiply-add
// by it stays an IMAD.WIDE): callers pass a kernel-argument-derived value.
__host__ __device__ __forceinline__ MixState mix_draw(const DrawKey& k, uint32_t d, uint32_t one) {
#ifdef __CUDA_ARCH__
  uint64_t x;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(x) : "r"(k.lo ^ d), "r"(one), "l"(k.addend));
#if MIX_MUL_PTX
  x = mul64_const(x ^ (x >> 30), 0x1CE4E5B9u, 0xBF58476Du);
  x = mul64_const(x ^ (x >> 27), 0x133111EBu, 0x94D049BBu);
#else
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
#endif
#else
  uint64_t x = (uint64_t)(k.lo ^ d) * one + k.addend;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
#endif
  return MixState{(uint32_t)x, (uint32_t)(x >> 32)};
}
// ---- chunk-constant form of splitmix64(pre ^ d) for d in one 512-coordinate
// chunk [cbase, cbase + 512) (cbase a multiple of 512).  With P = pre ^ cbase
// and j = d - cbase, pre ^ d = (P & ~511) + ((P & 511) ^ j) (disjoint bits),
// so the mixer input is z = Q + ((P & 511) ^ j) with Q = (P & ~511) + gamma.
// When lo32(Q) <= 2^32 - 512 that addition never carries: the high word of z
// is the chunk constant Q_hi, so is the high word of the first xorshift
// (Q_hi ^ (Q_hi >> 30)), and so is its share of the first product's high
// word.  Per coordinate the first two mixer steps then cost one add, one
// shift and one 3-input xor (low word only) and two multiply-adds.  A chunk
// whose Q_lo is within 512 of 2^32 (probability 2^-23 per key and chunk) is
// flagged not `fast` and takes the general draw (mix_draw).
struct ChunkDraw {
  uint32_t qe[4];  // Q_lo + ((p9 & 3) ^ e), e = 0..3
  uint64_t k2w;    // lo32((Q_hi ^ (Q_hi >> 30)) * lo32(C1)) << 32: the high word's share of
                   // y * lo32(C1), a 64-bit addend whose low word (0) the compiler cannot see
  uint32_t p9;     // P & 511, bit 31 set when the chunk is not `fast`
  uint32_t k1;     // Q_hi << 2: the high word's bits in lo32(z >> 30)
};
__host__ __device__ __forceinline__ ChunkDraw chunk_draw(uint64_t pre, uint32_t cbase) {
  const uint64_t P = pre ^ (uint64_t)cbase;
  const uint64_t Q = (P & ~511ull) + 0x9E3779B97F4A7C15ull;
  const uint32_t qlo = (uint32_t)Q, qhi = (uint32_t)(Q >> 32);
  const uint32_t p9 = (uint32_t)P & 511u;
  ChunkDraw k;
  for (uint32_t e = 0; e < 4; ++e) k.qe[e] = qlo + ((p9 & 3u) ^ e);
  k.k2w = (uint64_t)((qhi ^ (qhi >> 30)) * 0x1CE4E5B9u) << 32;
  k.p9 = p9 | (qlo <= 0xFFFFFE00u ? 0u : 0x80000000u);
  k.k1 = qhi << 2;
  return k;
}
__host__ __device__ __forceinline__ bool chunk_fast(const ChunkDraw& k) { return (k.p9 >> 31) == 0; }
// Low word of z for the lane's coordinate slice j = J0 + e (J0 a multiple of
// 4): (p9 ^ (J0 + e)) = ((p9 ^ J0) & ~3) + ((p9 & 3) ^ e), so
// zlo[e] = qe[e] + chunk_slice(k, J0).
__host__ __device__ __forceinline__ uint32_t chunk_slice(const ChunkDraw& k, uint32_t J0) {
  return (k.p9 ^ J0) & 0x1FCu;  // J0 < 512
}
// The mixer state (z before its final xorshift, as mix_draw) from zlo.
__host__ __device__ __forceinline__ MixState mix_chunk(const ChunkDraw& k, uint32_t zlo) {
  // y = z ^ (z >> 30): low word only (the high word is folded into k2)
  const uint32_t ylo = zlo ^ (zlo >> 30) ^ k.k1;
  // w = y * C1 mod 2^64
  const uint64_t w = (uint64_t)ylo * 0x1CE4E5B9u + k.k2w;
  const uint32_t wlo = (uint32_t)w;
  const uint32_t whi = (uint32_t)(w >> 32) + ylo * 0xBF58476Du;
  // v = w ^ (w >> 27)
#ifdef __CUDA_ARCH__
  const uint32_t vlo = wlo ^ __funnelshift_r(wlo, whi, 27);
#else
  const uint32_t vlo = wlo ^ (uint32_t)((((uint64_t)whi << 32) | wlo) >> 27);
#endif
  const uint32_t vhi = whi ^ (whi >> 27);
  // z = v * C2 mod 2^64
  const uint64_t z = (uint64_t)vlo * 0x133111EBu;
  const uint32_t zhi = (uint32_t)(z >> 32) + vlo * 0x94D049BBu + vhi * 0x133111EBu;
  return MixState{(uint32_t)z, zhi};
}

// Bits 11..42 and 43..63 of h = z ^ (z >> 31): lo32(h >> 11) and h_hi >> 11.
__host__ __device__ __forceinline__ uint32_t mant_lo(MixState z) {
#ifdef __CUDA_ARCH__
  return __funnelshift_r(z.lo, z.hi, 11) ^ (z.hi >> 10);
#else
  return (uint32_t)((((uint64_t)z.hi << 32) | z.lo) >> 11) ^ (z.hi >> 10);
#endif
}

// D1 = 1 + (m mod 2^52) 2^-52 in [1, 2) for m = h >> 11, built from the bits
// (no int -> fp conversion): mantissa = bits 11..62 of h.
__device__ __forceinline__ double unit_d1(uint64_t h) {
  const uint32_t hi = (uint32_t)(h >> 32);
  const uint32_t lo = __funnelshift_r((uint32_t)h, hi, 11);  // bits 11..42 of h
  const uint32_t mhi = (hi >> 11) & 0xFFFFFu;                 // bits 43..62 of h
  return __hiloint2double((int)(0x3FF00000u | mhi), (int)lo);
}

// rng.hpp:55-57: u = (h >> 11) * 2^-53.  With top = bit 63 of h and
// Dh = D1 / 2 in [0.5, 1) (same mantissa, exponent -1), u = Dh - (1 - top)/2:
// the subtraction is exact (Sterbenz), so u is bit-identical to the
// reference's value.  The constant is selected with integer ops.
__device__ __forceinline__ double unit_u53(uint64_t h) {
  const uint32_t hi = (uint32_t)(h >> 32);
  const uint32_t lo = __funnelshift_r((uint32_t)h, hi, 11);
  const uint32_t mhi = (hi >> 11) & 0xFFFFFu;
  const double dh = __hiloint2double((int)(0x3FE00000u | mhi), (int)lo);
  int32_t sgn;  // arithmetic shift kept as such (not a 64-bit compare + select)
  asm("shr.s32 %0, %1, 31;" : "=r"(sgn) : "r"(hi));
  const uint32_t c_hi = 0x3FE00000u & ~(uint32_t)sgn;  // top ? 0 : 0.5
  return __dsub_rn(dh, __hiloint2double((int)c_hi, 0));
}

// rng.hpp:60-65: lo + u * (hi - lo) (no contraction, same op order).
__device__ __forceinline__ double uniform_draw(uint64_t h, double lo,
                                               double hi) {
  return __dadd_rn(lo, __dmul_rn(unit_u53(h), __dsub_rn(hi, lo)));
}

// Round an in-box fp64 value to fp32 and keep it inside the fp32 image of
// the box [lo_f, hi_f] (the largest float interval inside [lower, upper]).
// Differs from a plain rounding only when rounding would leave the box.
__device__ __forceinline__ float to_f32_in_box(double x, float lo_f,
                                               float hi_f) {
  float f = __double2float_rn(x);
  f = f < lo_f ? lo_f : f;
  f = f > hi_f ? hi_f : f;
  return f;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sin^2(pi x): period 1, even, so with r = x - rint(x) in [-1/2, 1/2] it is
// (r P(r^2))^2 with P the degree-4 minimax fit of sin(pi r) / r (relative
// error 5e-9 in exact arithmetic, 1.8e-7 evaluated in fp32) — no quadrant
// logic, 7 FMA-pipe instructions instead of sinpif's ~25 (C4 explode).
__device__ __forceinline__ float sin_pi_sq(float x) {
  const float r = x - rintf(x);
  const float t = r * r;
  float p = fmaf(t, 0.07756161404419515f, -0.5982427027694103f);
  p = fmaf(t, p, 2.5500698108736963f);
  p = fmaf(t, p, -5.167709688780585f);
  p = fmaf(t, p, 3.141592636925161f);
  const float s = r * p;
  return s * s;
}

// Per-coordinate analytic terms; partial sums are fp32.
//   sphere     : x^2                                   (nets.cpp:80-84)
//   rastrigin  : x^2 + 20 sin^2(pi x)   == x^2 - 10 cos(2 pi x) + 10
//   ackley     : (x^2, cos 2 pi x = 1 - 2 sin^2(pi x))  two sums
__device__ __forceinline__ void analytic_terms(int kind, float x, float& s0,
                                               float& s1) {
  if (kind == OBJ_SPHERE) {
    s0 = fmaf(x, x, s0);
  } else if (kind == OBJ_RASTRIGIN) {
    s0 += fmaf(x, x, 20.0f * sin_pi_sq(x));
  } else {  // ackley
    s0 = fmaf(x, x, s0);
    s1 += fmaf(-2.0f, sin_pi_sq(x), 1.0f);
  }
}

// Final value from the (deterministically ordered) partial sums.
__device__ __forceinline__ float analytic_finalize(int kind, float s0,
                                                   float s1, uint64_t D) {
  if (kind == OBJ_ACKLEY) {
    const float inv = 1.0f / (float)D;
    return -20.0f * expf(-0.2f * sqrtf(s0 * inv)) - expf(s1 * inv) + 20.0f +
           2.718281828459045f;
  }
  return s0;
}

// Programmatic dependent launch (every engine kernel is launched with
// programmatic stream serialization, see pdl_launch): wait until the
// previous kernel has completed and its writes are visible; must precede
// any global access.  TRIGGER: first allow the next kernel in the stream to
// be scheduled now (used by the short latency-bound kernels only — an early
// trigger from the long kernels measured slower).
template <bool TRIGGER = false>
__device__ __forceinline__ void pdl_enter() {
  if (TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Launch with programmatic stream serialization: the launch (and block
// scheduling) of a kernel overlaps the tail of its predecessor; the kernel's
// pdl_enter() keeps the data dependency.  Works inside stream capture
// (programmatic graph edges).  MGFWA_PDL=0 disables it.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("MGFWA_PDL");
    return e == nullptr || e[0] != '0';
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace mgfwa_b200
