// k_engine.cu — the MGFWA generation kernels (everything except the tensor-
// core NN fitness, which lives in k_mlp_tc.cu).
//
// One generation = the body of run()'s loop, engine.cpp:359-417:
//   (population_range, engine.cpp:22-41, is computed by the previous
//    generation's tail kernel k_record_copy)
//   k_explode_map    explode + random_mapping    engine.cpp:78-131 (+ fused
//                    analytic fitness partials, + bf16 shadow for NN)
//   [NN fitness]     batched_apply(sparks)       backend.cpp:28-67
//   k_rank           finalize spark fitness (NaN->+inf, backend.cpp:15-24)
//                    + stable (fitness, index) ranking, engine.cpp:151-157
//   k_guides         guiding_vector + multi_guiding_sparks + random_mapping
//                    (kGuide), engine.cpp:133-196 (+ fused partials)
//   [NN fitness]     batched_apply(guides)
//   k_select         finalize guide fitness + select_best argmin +
//                    update_amplitudes + winner row copy, engine.cpp:198-256
//   k_loser          loser_out decision, engine.cpp:258-286, 394-410
//   k_fresh_rows     loser reinit rows (kReinit), engine.cpp:287-294
//   [NN fitness]     batched_apply(losers)
//   k_finalize_record loser fitness commit + record_wave, engine.cpp:340-351
//   k_record_copy    best-position copy on strict improvement +
//                    population_range of the next generation
// All kernels read ctl->active / ctl->iteration from HBM so that one CUDA
// graph replays every generation unchanged.
#include "common.cuh"
#include "engine_view.cuh"
#include "kernels.h"

namespace mgfwa_b200 {

namespace {

constexpr int kWarps = 8;  // warps per block for the work-item kernels

// Counter for NaN evaluations of work only this shard does (Ctl::nan_own).
__device__ __forceinline__ unsigned long long* nan_counter_own(const EngineView& v) {
  return (unsigned long long*)(v.nan_mode ? &v.ctl->nan_own : &v.ctl->nan_count);
}

__device__ __forceinline__ bool gen_inactive(const EngineView& v) {
  return *(volatile int*)&v.ctl->active == 0;
}

// Partial sums of one row -> fitness (fp32), NaN -> +inf (backend.cpp:15-24).
// One fixed order per run, whichever kernel finalizes, so a candidate's
// cached fitness and its re-evaluation are bit-identical:
//   nparts <= kSeqParts (the tensor-core objectives: one partial per 128
//   samples; D <= 8192 analytic rows): ((p0 + p1) + p2) + ... in one thread
//   (row_sums_seq) — no shuffles, so a finalizing thread per row is cheap;
//   larger nparts (the 512-coordinate chunks of long analytic rows):
//   lane-strided sums and a butterfly over the warp.
constexpr uint32_t kSeqParts = 16;

__device__ __forceinline__ float2 row_sums_seq(const EngineView& v, const float* part, uint64_t row) {
  const float2* p = reinterpret_cast<const float2*>(part + row * (uint64_t)v.nparts * 2);
  float a = 0.0f, b = 0.0f;
  for (uint32_t c = 0; c < v.nparts; ++c) {
    const float2 q = p[c];
    a += q.x;
    b += q.y;
  }
  return make_float2(a, b);
}

__device__ __forceinline__ float finalize_value(const EngineView& v, float a, float b, bool* was_nan) {
  const float f = v.nn ? a / (float)v.samples : analytic_finalize(v.obj_kind, a, b, v.D);
  *was_nan = isnan(f);
  return isnan(f) ? __int_as_float(0x7f800000) : f;
}

// Warp-cooperative form (all 32 lanes call it and get every row's value):
// R rows at once (their loads in flight together); rows[r] < 0 are skipped.
template <int R>
__device__ __forceinline__ void finalize_rows(const EngineView& v, const float* part,
                                              const int64_t (&rows)[R], float (&out)[R],
                                              unsigned& nan_count) {
  const int lane = threadIdx.x & 31;
  float s0[R], s1[R];
  const bool seq = v.nparts <= kSeqParts;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    s0[r] = s1[r] = 0.0f;
    if (rows[r] < 0) continue;
    if (seq) {  // every lane: the same sequential sums (broadcast loads)
      const float2 q = row_sums_seq(v, part, (uint64_t)rows[r]);
      s0[r] = q.x, s1[r] = q.y;
      continue;
    }
    const float* p = part + (uint64_t)rows[r] * (uint64_t)v.nparts * 2;
    for (uint32_t c = lane; c < v.nparts; c += 32) {
      s0[r] += p[2 * c];
      s1[r] += p[2 * c + 1];
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const float a = seq ? s0[r] : __shfl_sync(0xffffffffu, warp_sum(s0[r]), 0);
    const float b = seq ? s1[r] : __shfl_sync(0xffffffffu, warp_sum(s1[r]), 0);
    bool nan;
    out[r] = finalize_value(v, a, b, &nan);
    nan_count += nan && rows[r] >= 0;
  }
}

__device__ __forceinline__ float finalize_row(const EngineView& v,
                                              const float* part, uint64_t row,
                                              bool* was_nan) {
  const int64_t rows[1] = {(int64_t)row};
  float out[1];
  unsigned n = 0;
  finalize_rows<1>(v, part, rows, out, n);
  *was_nan = n != 0;
  return out[0];
}

// Random-mapping repair of one coordinate (engine.cpp:119-125):
// out-of-box (inclusive test, config.hpp:22-24) -> U[pop_lo, pop_hi).
__device__ __forceinline__ float map_coord(const EngineView& v, double x,
                                           uint64_t d, uint64_t map_prefix,
                                           const float* plo, const float* phi) {
  if (!(x >= v.lower[d] && x <= v.upper[d])) {
    x = uniform_draw(splitmix64(map_prefix ^ d), (double)plo[d], (double)phi[d]);
  }
  return to_f32_in_box(x, v.lower_f[d], v.upper_f[d]);
}

__device__ __forceinline__ void store_row4(float* dst, __nv_bfloat16* dst_h,
                                           uint64_t off, const float (&x)[4]) {
  *reinterpret_cast<float4*>(dst + off) = make_float4(x[0], x[1], x[2], x[3]);
  if (dst_h != nullptr) {
    __nv_bfloat162 a = __floats2bfloat162_rn(x[0], x[1]);
    __nv_bfloat162 b = __floats2bfloat162_rn(x[2], x[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(dst_h + off) = u;
  }
}

__device__ __forceinline__ void store_bf16x4(__nv_bfloat16* dst_h, uint64_t off,
                                             const float (&x)[4]) {
  __nv_bfloat162 a = __floats2bfloat162_rn(x[0], x[1]);
  __nv_bfloat162 b = __floats2bfloat162_rn(x[2], x[3]);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(dst_h + off) = u;
}

}  // namespace

// ------------------------------------------------------------------ range
// population_range, engine.cpp:22-41 (std::min/std::max keep-first order).
__global__ void k_pop_range(EngineView v) {
  pdl_enter();
  if (gen_inactive(v)) return;
  const uint64_t total = v.B * v.D;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = i / v.D, d = i % v.D;
    const float* p = v.pos + (b * v.mu) * v.Dp + d;
    float mn = p[0], mx = p[0];
    for (uint64_t n = 1; n < v.mu; ++n) {
      const float x = p[n * v.Dp];
      mn = (x < mn) ? x : mn;
      mx = (mx < x) ? x : mx;
    }
    v.pop_lo[b * v.Dp + d] = mn;
    v.pop_hi[b * v.Dp + d] = mx;
  }
}

// ---------------------------------------------------------------- explode
// explode (engine.cpp:78-101) fused with random_mapping(kMapping)
// (engine.cpp:103-131), the fp32 store, the bf16 shadow (NN) and the
// analytic fitness partial sums.
//
// Work item = (firework, group of kSparkGroup sparks, 512-coordinate chunk):
// the firework row, the box images and the pos -> fp64 conversions are
// loaded once and reused by the sparks of the group.  Per coordinate the
// cost is one splitmix64 round (hoisted key prefix), an exact bit-built
// t = -1 + 2u (no int->fp conversion), one DMUL + DADD in fp64 and one
// rounding to fp32.  The in-box test runs on the rounded float against the
// fp32 box images (exact whenever strictly inside, see in_box_fast).  The
// remaining coordinates — out of the box (random mapping) or on the 1-ulp
// boundary — are finished in place: whenever any lane of the warp has one
// among a spark's 4 coordinates, the warp runs the exact test and the
// kMapping draw for those 4 coordinates as 4 independent chains and selects
// per lane.  Out-of-box coordinates are common (C2: 35% of them once the
// amplitudes reach the range, so nearly every warp has one in every spark
// slice); this dense form beats every compaction variant measured.
#ifndef EXPLODE_KG
#define EXPLODE_KG 4
#endif
constexpr int kSparkGroup = EXPLODE_KG;

// t = -1 + u * 2 for u = (h >> 11) * 2^-53, exactly as the reference's
// uniform_sample(key, -1, 1) (rng.hpp:55-65): with m = h >> 11 and
// D1 = 1 + (m mod 2^52) 2^-52 in [1, 2), t = D1 - (2 - (m >> 52)); both
// subtractions are exact (Sterbenz), so t is bit-identical to the fp64
// reference value without an int -> fp conversion.
__device__ __forceinline__ double unit_pm1(uint64_t h) {
  const uint32_t hi = (uint32_t)(h >> 32);
  const uint32_t c_hi = 0x40000000u - ((hi >> 11) & 0x100000u);  // top ? 1.0 : 2.0
  return __dsub_rn(unit_d1(h), __hiloint2double((int)c_hi, 0));
}

// unit_pm1 / unit_u53 of h = splitmix64(pre ^ d) from the mixer state (see
// mix_draw): bit-identical, three ALU instructions fewer per draw.
// Logical right shifts as mul.hi(x, 2^(32-k)) with an opaque multiplier:
// IMAD.HI on the FMA pipe instead of SHF on the ALU pipe.  Level 0: none;
// 1: the mantissa shifts of the draws; 2: also the mixer's xorshifts.
#ifndef EXPLODE_IMAD_SHR
#define EXPLODE_IMAD_SHR 0
#endif
__device__ __forceinline__ uint32_t shr_fma(uint32_t x, uint32_t pow2) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(pow2));
  return r;
}
template <int K>
__device__ __forceinline__ uint32_t shr_k(uint32_t x, uint32_t one, int level) {
  return level ? shr_fma(x, one << (32 - K)) : x >> K;
}
// mix_chunk (common.cuh) with the xorshifts' shifts on the FMA pipe at level 2.
__device__ __forceinline__ MixState mix_chunk_k(const ChunkDraw& k, uint32_t zlo, uint32_t one) {
  constexpr int L = EXPLODE_IMAD_SHR >= 2;
  const uint32_t ylo = zlo ^ shr_k<30>(zlo, one, L) ^ k.k1;
  const uint64_t w = (uint64_t)ylo * 0x1CE4E5B9u + k.k2w;
  const uint32_t wlo = (uint32_t)w;
  const uint32_t whi = (uint32_t)(w >> 32) + ylo * 0xBF58476Du;
  const uint32_t vlo = wlo ^ __funnelshift_r(wlo, whi, 27);
  const uint32_t vhi = whi ^ shr_k<27>(whi, one, L);
  const uint64_t z = (uint64_t)vlo * 0x133111EBu;
  const uint32_t zhi = (uint32_t)(z >> 32) + vlo * 0x94D049BBu + vhi * 0x133111EBu;
  return MixState{(uint32_t)z, zhi};
}
// D1 = 1 + (m mod 2^52) 2^-52 of h = z ^ (z >> 31), m = h >> 11 (mant_lo,
// common.cuh): the top bit of z.hi >> 11 (bit 20) is absorbed by the exponent
// bits of 1.0.
__device__ __forceinline__ double draw_d1(MixState z, uint32_t one) {
  constexpr int L = EXPLODE_IMAD_SHR >= 1;
  const uint32_t lo = __funnelshift_r(z.lo, z.hi, 11) ^ shr_k<10>(z.hi, one, L);
  return __hiloint2double((int)(0x3FF00000u | shr_k<11>(z.hi, one, L)), (int)lo);
}

// `one` = 1, opaque to the compiler: the sign mask s = (z.hi < 0 ? -1 : 0)
// is mul.hi(z.hi, one), an IMAD.HI on the FMA pipe instead of a shift on the
// (saturated) ALU pipe.
__device__ __forceinline__ int32_t sign_mask(uint32_t x, uint32_t one) {
  int32_t s;
  asm("mul.hi.s32 %0, %1, %2;" : "=r"(s) : "r"(x), "r"(one));
  return s;
}
__device__ __forceinline__ double unit_pm1_z(MixState z, uint32_t one) {
  // t = D1 - (top ? 1 : 2), exact
  const double d1 = draw_d1(z, one);
  const uint32_t s = (uint32_t)sign_mask(z.hi, one);
  const uint32_t c_hi = (s & 0x3FF00000u) | (~s & 0x40000000u);  // top ? 1.0 : 2.0
  return __dsub_rn(d1, __hiloint2double((int)c_hi, 0));
}
// 2u = D1 - (top ? 0 : 1) for u = (h >> 11) 2^-53 (exact); the caller
// multiplies by half the interval width (exact scaling), so
// lo + u * w == lo + unit_2u_z(z) * (w / 2) bit for bit.
__device__ __forceinline__ double unit_2u_z(MixState z, uint32_t one) {
  const double d1 = draw_d1(z, one);
  const uint32_t s = (uint32_t)sign_mask(z.hi, one);
  return __dsub_rn(d1, __hiloint2double((int)(~s & 0x3FF00000u), 0));
}

// Exact in-box test for x = round_f32(s): strictly between the fp32 box
// images implies lower <= s <= upper (lo_f >= lower, and s > lo_f because
// s rounds to a float above lo_f); callers fall back to the exact test
// otherwise.
__device__ __forceinline__ bool in_box_fast(float x, float lo_f, float hi_f) {
  return x > lo_f && x < hi_f;
}

// rng.hpp:43-49 absorbed up to the iteration for the explode and mapping
// streams: (x, y) = key prefixes of (seed, kExplode, it) and (seed, kMapping, it).
__device__ __forceinline__ ulonglong2 explode_stream_prefixes(const EngineView& v) {
  const uint64_t it = v.ctl->iteration;
  const uint64_t hs = splitmix64(v.seed);
  return make_ulonglong2(splitmix64(splitmix64(hs ^ kExplode) ^ it), splitmix64(splitmix64(hs ^ kMapping) ^ it));
}

// Dynamic shared memory of k_explode_map: the block's 512-coordinate chunk
// of the box (fp64 and its fp32 images) and of the population range,
// staged once per work item, plus the per-warp key prefixes.
struct ExplodeChunk {
  double lo[kChunk], hi[kChunk];
  double plo[kChunk], pw[kChunk];  // pop_lo and (pop_hi - pop_lo) / 2 in fp64
  float lof[kChunk], hif[kChunk];
};
#ifndef EXPLODE_SMEM_KEYS
#define EXPLODE_SMEM_KEYS 1  // draw keys in shared memory: 80 registers, 3 blocks/SM, no spills (C2 explode 157 -> 156.6 us; in registers at 3 blocks/SM it spills: 172 us)
#endif
#ifndef EXPLODE_STCS
#define EXPLODE_STCS 1  // fp32 spark rows of NN objectives stored with the evict-first hint (C2 0.2710 -> 0.2679 ms)
#endif
#ifndef EXPLODE_MINB
#define EXPLODE_MINB 3  // blocks per SM the main explode kernel is compiled for
#endif
struct ExplodeWarp {
  uint64_t pre[2 * kSparkGroup];  // explode / mapping key prefixes
  DrawKey keys[2 * kSparkGroup];  // their draw keys (EXPLODE_SMEM_KEYS)
  ChunkDraw ck[2 * kSparkGroup];  // their chunk-constant draws for the current chunk
};
constexpr size_t kExplodeSmem = sizeof(ExplodeChunk) + kWarps * sizeof(ExplodeWarp);

// One 128-coordinate slice of kSparkGroup sparks.  FULL: every spark of the
// group exists and the slice lies inside [0, D) (no per-element guards).
// CHUNK: draws from the chunk-constant form (ck, every key of the group
// `fast` in this chunk); otherwise from the general draw keys (pe, pm).
template <int KIND, bool FULL, bool CHUNK, int KG = kSparkGroup>
__device__ __forceinline__ void explode_slice(const EngineView& v, const ExplodeChunk& ch,
                                              int lane, uint32_t cbase, uint32_t qoff,
                                              uint64_t f, uint64_t k0, int kn, double a,
                                              const DrawKey* pe, const DrawKey* pm,
                                              const ChunkDraw* ck, uint32_t one,
                                              float (&s0)[KG], float (&s1)[KG]) {
  const uint32_t D = (uint32_t)v.D;
  const uint32_t li0 = qoff + lane * 4;  // index inside the staged chunk
  const uint32_t d0 = cbase + li0;
  const bool on = FULL || d0 < D;
  const int nvalid = FULL ? 4 : (on ? (D - d0 < 4 ? (int)(D - d0) : 4) : 0);
  float4 p4 = make_float4(0.f, 0.f, 0.f, 0.f);
  if (on) p4 = *reinterpret_cast<const float4*>(v.pos + f * v.Dp + d0);
  const float4 lf4 = *reinterpret_cast<const float4*>(&ch.lof[li0]);
  const float4 uf4 = *reinterpret_cast<const float4*>(&ch.hif[li0]);
  const double pd[4] = {(double)p4.x, (double)p4.y, (double)p4.z, (double)p4.w};
  const float lf[4] = {lf4.x, lf4.y, lf4.z, lf4.w};
  const float uf[4] = {uf4.x, uf4.y, uf4.z, uf4.w};
#pragma unroll
  for (int kk = 0; kk < KG; ++kk) {
    if (!FULL && kk >= kn) break;
    float x[4];
    double sv[4];
    unsigned slow = 0;
    MixState ze[4];
    if constexpr (CHUNK) {
      const ChunkDraw& kc = ck[kk];
      const uint32_t tj = chunk_slice(kc, li0);
#pragma unroll
      for (int e = 0; e < 4; ++e) ze[e] = mix_chunk_k(kc, kc.qe[e] + tj, one);
    } else {
      const DrawKey ke = pe[kk];
#pragma unroll
      for (int e = 0; e < 4; ++e) ze[e] = mix_draw(ke, d0 + e, one);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      sv[e] = __dadd_rn(pd[e], __dmul_rn(unit_pm1_z(ze[e], one), a));
      x[e] = __double2float_rn(sv[e]);
      const bool need = !in_box_fast(x[e], lf[e], uf[e]);
      if (FULL ? need : (e < nvalid && need)) slow |= 1u << e;
    }
    // Out-of-box / boundary coordinates of this spark: exact inclusive test
    // (config.hpp:22-24) and the kMapping draw U[pop_lo, pop_hi)
    // (engine.cpp:119-125), 4 independent chains, selected per lane.
    if (__any_sync(0xffffffffu, slow != 0)) {
      const double2 lo01 = *reinterpret_cast<const double2*>(&ch.lo[li0]);
      const double2 lo23 = *reinterpret_cast<const double2*>(&ch.lo[li0 + 2]);
      const double2 hi01 = *reinterpret_cast<const double2*>(&ch.hi[li0]);
      const double2 hi23 = *reinterpret_cast<const double2*>(&ch.hi[li0 + 2]);
      const double2 pl01 = *reinterpret_cast<const double2*>(&ch.plo[li0]);
      const double2 pl23 = *reinterpret_cast<const double2*>(&ch.plo[li0 + 2]);
      const double2 pw01 = *reinterpret_cast<const double2*>(&ch.pw[li0]);
      const double2 pw23 = *reinterpret_cast<const double2*>(&ch.pw[li0 + 2]);
      const double lo[4] = {lo01.x, lo01.y, lo23.x, lo23.y};
      const double hi[4] = {hi01.x, hi01.y, hi23.x, hi23.y};
      const double pl[4] = {pl01.x, pl01.y, pl23.x, pl23.y};
      const double pw[4] = {pw01.x, pw01.y, pw23.x, pw23.y};
      MixState zm[4];
      if constexpr (CHUNK) {
        const ChunkDraw& kc = ck[KG + kk];
        const uint32_t tj = chunk_slice(kc, li0);
#pragma unroll
        for (int e = 0; e < 4; ++e) zm[e] = mix_chunk_k(kc, kc.qe[e] + tj, one);
      } else {
        const DrawKey km = pm[kk];
#pragma unroll
        for (int e = 0; e < 4; ++e) zm[e] = mix_draw(km, d0 + e, one);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double u = unit_2u_z(zm[e], one);  // 2u; pw holds half the width
        const float m = __double2float_rn(__dadd_rn(pl[e], __dmul_rn(u, pw[e])));
        const float r = (sv[e] >= lo[e] && sv[e] <= hi[e]) ? x[e] : m;
        x[e] = ((slow >> e) & 1u) ? fminf(fmaxf(r, lf[e]), uf[e]) : x[e];
      }
    }
    if (on) {
      if (!FULL) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e >= nvalid) x[e] = 0.0f;
      }
      if (KIND != 0) {
        float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (FULL || e < nvalid) analytic_terms(KIND, x[e], a0, a1);
        s0[kk] += a0;
        s1[kk] += a1;
      }
      const uint64_t off = ((f - v.f_lo) * v.lam + k0 + kk) * v.Dp + d0;  // local spark row
#if EXPLODE_STCS
      // NN objective: the fp32 rows (read back only for the ranked / winning
      // sparks) stream past L2 (evict-first) so the bf16 shadow the tcgen05
      // fitness reads next stays L2-resident
      if (KIND == 0)
        __stcs(reinterpret_cast<float4*>(v.sparks + off), make_float4(x[0], x[1], x[2], x[3]));
      else
#endif
        *reinterpret_cast<float4*>(v.sparks + off) = make_float4(x[0], x[1], x[2], x[3]);
      if (KIND == 0) store_bf16x4(v.sparks_h, off, x);
    }
  }
}

// One warp: spark group g (kSparkGroup sparks) of local firework fl over the
// staged chunk c (box images + population range of the firework's batch).
template <int KIND, int KG = kSparkGroup>
__device__ __forceinline__ void explode_group(const EngineView& v, const ExplodeChunk& ch,
                                              ExplodeWarp& wq, int lane, uint32_t c, uint64_t fl,
                                              uint64_t g, ulonglong2 hs) {
  static_assert(KG <= kSparkGroup, "ExplodeWarp holds kSparkGroup keys per stream");
  const uint32_t D = (uint32_t)v.D;
  const uint64_t f = v.f_lo + fl;
  const uint64_t b = f / v.mu, n = f % v.mu;
  const uint32_t cbase = c * kChunk;
  const uint64_t k0 = g * KG;
  const int kn = (int)(v.lam - k0 < (uint64_t)KG ? v.lam - k0 : KG);
  // key prefixes: lanes [0, KG) explode, [KG, 2KG) mapping (hoisted
  // rng.hpp:43-51 up to field k; each draw is then one splitmix64 round).
  // hs = the (seed, stream, iteration) part, computed once per launch.
  {
    const bool ex = lane < KG;
    const int kl = ex ? lane : lane - KG;
    if (lane < 2 * KG && kl < kn) {
      uint64_t h = splitmix64((ex ? hs.x : hs.y) ^ b);
      h = splitmix64(h ^ n);
      wq.pre[lane] = splitmix64(h ^ (k0 + (uint64_t)kl));
    }
  }
  __syncwarp();
  // chunk-constant draws of this chunk; the general keys serve a group with
  // any key near a carry boundary (2^-23 per key and chunk)
  bool fast_key = true;
  if (lane < 2 * KG) {
    wq.ck[lane] = chunk_draw(wq.pre[lane], cbase);
    fast_key = chunk_fast(wq.ck[lane]);
  }
  const bool fast = __all_sync(0xffffffffu, fast_key) && !v.explode_general;
#if EXPLODE_SMEM_KEYS
  if (lane < 2 * KG) wq.keys[lane] = draw_key(wq.pre[lane]);
  __syncwarp();
  const DrawKey* pe = wq.keys;
  const DrawKey* pm = wq.keys + KG;
#else
  DrawKey pe[KG], pm[KG];
#pragma unroll
  for (int kk = 0; kk < KG; ++kk) {
    pe[kk] = draw_key(wq.pre[kk]);
    pm[kk] = draw_key(wq.pre[KG + kk]);
  }
  __syncwarp();  // wq.pre is reused by this warp's next group
#endif
  const uint32_t one = (uint32_t)(v.Dp != 0);  // 1, opaque to the compiler (see mix_draw)
  const double a = v.amp[f];
  float s0[KG], s1[KG];
#pragma unroll
  for (int kk = 0; kk < KG; ++kk) s0[kk] = s1[kk] = 0.0f;
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    const uint32_t qoff = q * 128;
    if (cbase + qoff >= D) break;  // warp-uniform
    if (!fast)
      explode_slice<KIND, false, false, KG>(v, ch, lane, cbase, qoff, f, k0, kn, a, pe, pm, wq.ck, one, s0, s1);
    else if (kn == KG && cbase + qoff + 128 <= D)
      explode_slice<KIND, true, true, KG>(v, ch, lane, cbase, qoff, f, k0, kn, a, pe, pm, wq.ck, one, s0, s1);
    else
      explode_slice<KIND, false, true, KG>(v, ch, lane, cbase, qoff, f, k0, kn, a, pe, pm, wq.ck, one, s0, s1);
  }
#if EXPLODE_SMEM_KEYS
  __syncwarp();  // wq.keys are reused by this warp's next group
#endif
  if (KIND != 0) {
#pragma unroll
    for (int kk = 0; kk < KG; ++kk) {
      if (kk >= kn) break;
      const float t0 = warp_sum(s0[kk]);
      const float t1 = warp_sum(s1[kk]);
      if (lane == 0) {
        const uint64_t r = fl * v.lam + k0 + kk;
        v.spart[(r * v.nparts + c) * 2] = t0;
        v.spart[(r * v.nparts + c) * 2 + 1] = t1;
      }
    }
  }
}

// Stage chunk c of batch b: box (fp64 and fp32 images) and population range.
__device__ __forceinline__ void stage_explode_chunk(const EngineView& v, ExplodeChunk& ch,
                                                    uint64_t b, uint32_t c) {
  const uint32_t D = (uint32_t)v.D;
  const uint32_t cbase = c * kChunk;
  for (uint32_t i = threadIdx.x; i < kChunk; i += blockDim.x) {
    const uint32_t d = cbase + i;
    const bool in = d < D;
    ch.lo[i] = in ? v.lower[d] : 0.0;
    ch.hi[i] = in ? v.upper[d] : 0.0;
    ch.lof[i] = in ? v.lower_f[d] : 0.0f;
    ch.hif[i] = in ? v.upper_f[d] : 0.0f;
    const double pl = in ? (double)v.pop_lo[b * v.Dp + d] : 0.0;
    const double ph = in ? (double)v.pop_hi[b * v.Dp + d] : 0.0;
    ch.plo[i] = pl;
    ch.pw[i] = 0.5 * __dsub_rn(ph, pl);  // half the width (see unit_2u_z)
  }
}

// Work item = (firework f, 512-coordinate chunk c, 8 consecutive spark
// groups): the block stages the chunk's box / population range once; warp w
// takes spark group 8*item_group + w.
// KIND == 0: NN objective (bf16 shadow, no analytic partials); otherwise the
// analytic objective kind whose partial sums are fused in.
// MINB = 3 (the chunk variant run beside the persistent tcgen05 fitness
// kernel): <= 85 registers so one 256-thread block fits next to the MLP CTA's
// 384 threads on the same SM.
template <int KIND, int MINB = 2>
__global__ void __launch_bounds__(256, MINB) k_explode_map(EngineView v) {
  pdl_enter();
  if (gen_inactive(v)) return;
  constexpr int KG = kSparkGroup;
  extern __shared__ __align__(16) uint8_t ex_smem[];
  ExplodeChunk& ch = *reinterpret_cast<ExplodeChunk*>(ex_smem);
  ExplodeWarp* wqs = reinterpret_cast<ExplodeWarp*>(ex_smem + sizeof(ExplodeChunk));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ExplodeWarp& wq = wqs[warp];
  const uint64_t ngrp = (v.lam + KG - 1) / KG;
  const uint64_t nsup = (ngrp + kWarps - 1) / kWarps;  // groups of 8 spark groups
  const uint64_t items = v.Fl * v.nch * nsup;
  const ulonglong2 hs = explode_stream_prefixes(v);
  for (uint64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const uint64_t sup = item % nsup, rest = item / nsup;
    const uint32_t c = (uint32_t)(rest % v.nch);
    const uint64_t fl = rest / v.nch, b = (v.f_lo + fl) / v.mu;
    __syncthreads();  // previous item's readers are done with the chunk
    stage_explode_chunk(v, ch, b, c);
    __syncthreads();
    const uint64_t g = sup * kWarps + warp;
    if (g >= ngrp) continue;  // warp-uniform
    explode_group<KIND>(v, ch, wq, lane, c, fl, g, hs);
  }
}

static unsigned explode_blocks(const EngineView& v, int nsm) {
  const uint64_t ngrp = (v.lam + kSparkGroup - 1) / kSparkGroup;
  const uint64_t items = v.Fl * v.nch * ((ngrp + kWarps - 1) / kWarps);
#ifndef EXPLODE_CAP_MULT
#define EXPLODE_CAP_MULT 256  // blocks per SM cap (measured: 8 -> 256 is 4% faster on C2, C3, C5: finer tail)
#endif
  const uint64_t cap = (uint64_t)nsm * EXPLODE_CAP_MULT;
  return (unsigned)(items < cap ? items : cap);
}

template <int KIND>
static void explode_launch_k(const EngineView& v, unsigned grid, cudaStream_t s) {
  pdl_launch(k_explode_map<KIND, EXPLODE_MINB>, grid, 256, kExplodeSmem, s, v);
}

#ifndef RANK_THREADS
#define RANK_THREADS 1024
#endif
constexpr int kRankThreads = RANK_THREADS;
constexpr int kRankSmemMax = (int)(kMaxSparksPerFirework * sizeof(uint64_t));
__global__ void __launch_bounds__(kRankThreads) k_rank(EngineView v);

cudaError_t prepare_engine_kernels() {
  cudaError_t e = cudaSuccess;
  const int bytes = (int)kExplodeSmem;
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_explode_map<0, EXPLODE_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_explode_map<0, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_explode_map<OBJ_SPHERE, EXPLODE_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_explode_map<OBJ_RASTRIGIN, EXPLODE_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_explode_map<OBJ_ACKLEY, EXPLODE_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, kRankSmemMax);
  return e;
}

// Explode + mapping of the owned fireworks [f0, f0 + nf) only (the spark
// rows of that range), in the register-capped variant that co-resides with
// the tcgen05 fitness kernel: the pipelined NN generation runs the fitness of
// firework chunk c while chunk c + 1 explodes.
void launch_explode_fireworks(const EngineView& v, uint64_t f0, uint64_t nf, int nsm, cudaStream_t s) {
  EngineView c = v;
  c.f_lo = v.f_lo + f0;
  c.Fl = nf;
  c.sparks = v.sparks + f0 * v.lam * v.Dp;
  if (v.sparks_h) c.sparks_h = v.sparks_h + f0 * v.lam * v.Dp;
  pdl_launch(k_explode_map<0, 3>, explode_blocks(c, nsm), 256, kExplodeSmem, s, c);
}

static void launch_explode_map_impl(const EngineView& v, int nsm, cudaStream_t s) {
  const unsigned grid = explode_blocks(v, nsm);
  const int kind = v.nn ? 0 : v.obj_kind;
  switch (kind) {
    case 0: explode_launch_k<0>(v, grid, s); break;
    case OBJ_SPHERE: explode_launch_k<OBJ_SPHERE>(v, grid, s); break;
    case OBJ_RASTRIGIN: explode_launch_k<OBJ_RASTRIGIN>(v, grid, s); break;
    default: explode_launch_k<OBJ_ACKLEY>(v, grid, s); break;
  }
}

// ------------------------------------------------------------------- rank
// Finalize spark fitness, then the stable ranking of guiding_vector
// (engine.cpp:151-157): order by (fitness asc, index asc); record the top
// `top` indices (best first) and the bottom `top` (rank order).
// One block per firework.
// Total-order key of (fitness asc, index asc): -0.0 == +0.0 as in the
// reference's comparator (fi != fj is false for them), so -0 is canonicalised.
__device__ __forceinline__ uint64_t rank_key(float x, uint32_t k) {
  uint32_t u = __float_as_uint(x == 0.0f ? 0.0f : x);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((uint64_t)u << 32) | k;
}

#ifndef RANK_TRIGGER
#define RANK_TRIGGER 0  // measured: no early trigger is 1.5 us faster per C2 generation
#endif
__global__ void __launch_bounds__(kRankThreads) k_rank(EngineView v) {
  pdl_enter<RANK_TRIGGER != 0>();
  if (gen_inactive(v)) return;
  extern __shared__ uint64_t keys[];  // [lambda] sort keys, then [lambda] rank counts (split counting)
  const uint64_t fl = blockIdx.x;     // local firework
  const uint32_t lam = (uint32_t)v.lam;
  if (threadIdx.x == 0) v.fit_prev[v.f_lo + fl] = v.fit[v.f_lo + fl];  // for k_select's parts
  unsigned nan_local = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  if (v.nparts <= kSeqParts || v.injected_fitness) {
    // one thread per spark row (sequential partial sums, see finalize_rows)
    for (uint32_t k = threadIdx.x; k < lam; k += blockDim.x) {
      const uint64_t row = fl * lam + k;
      float x;
      if (v.injected_fitness) {
        x = v.sfit[row];
      } else {
        const float2 q = row_sums_seq(v, v.spart, row);
        bool nan;
        x = finalize_value(v, q.x, q.y, &nan);
        nan_local += nan;
        v.sfit[row] = x;
      }
      keys[k] = rank_key(x, k);
    }
    nan_local = __reduce_add_sync(0xffffffffu, nan_local);
  } else {
    constexpr int R = 4;  // rows per warp step (their loads in flight together)
    for (uint32_t k0 = warp * R; k0 < lam; k0 += nwarp * R) {
      int64_t rows[R];
      float x[R];
#pragma unroll
      for (int r = 0; r < R; ++r) rows[r] = (k0 + r < lam) ? (int64_t)(fl * lam + k0 + r) : -1;
      finalize_rows<R>(v, v.spart, rows, x, nan_local);
      float xl = x[0];
      int64_t rl = rows[0];
#pragma unroll
      for (int r = 1; r < R; ++r) {
        xl = lane == r ? x[r] : xl;
        rl = lane == r ? rows[r] : rl;
      }
      if (lane < R && rl >= 0) {
        v.sfit[rl] = xl;
        keys[k0 + lane] = rank_key(xl, k0 + lane);
      }
    }
  }
  if (lane == 0 && nan_local) atomicAdd(nan_counter_own(v), (unsigned long long)nan_local);
  if (v.M == 0) return;
  __syncthreads();
  // Rank by counting: keys are a total order with distinct values, so
  // rank(k) = #{j : key_j < key_k} is the position std::sort with the
  // reference comparator (engine.cpp:152-157) gives spark k.  All threads
  // read the same key_j at once (shared-memory broadcast).  With room for
  // P >= 2 threads per spark, the j range is split P ways and the partial
  // counts summed in shared memory.
  const uint32_t top = (uint32_t)v.top;
  int* out = v.rank_idx + fl * 2 * top;
  const uint32_t P = lam * 2 <= blockDim.x && lam * 12 <= kRankSmemMax ? blockDim.x / lam : 1u;
  if (P >= 2) {
    uint32_t* cnt = reinterpret_cast<uint32_t*>(keys + ((lam + 1) & ~1u));
    for (uint32_t k = threadIdx.x; k < lam; k += blockDim.x) cnt[k] = 0;
    __syncthreads();
    const uint32_t k = threadIdx.x % lam, p = threadIdx.x / lam;
    if (p < P) {
      const uint64_t kk = keys[k];
      const uint32_t j0 = lam * p / P, j1 = lam * (p + 1) / P;
      uint32_t r0 = 0, r1 = 0, j = j0;
      for (; j + 2 <= j1; j += 2) {
        r0 += keys[j] < kk;
        r1 += keys[j + 1] < kk;
      }
      if (j < j1) r0 += keys[j] < kk;
      atomicAdd(&cnt[k], r0 + r1);
    }
    __syncthreads();
    for (uint32_t k2 = threadIdx.x; k2 < lam; k2 += blockDim.x) {
      const uint32_t r = cnt[k2];
      if (r < top) out[r] = (int)k2;
      if (r >= lam - top) out[top + (r - (lam - top))] = (int)k2;
    }
    return;
  }
  for (uint32_t k = threadIdx.x; k < lam; k += blockDim.x) {
    const uint64_t kk = keys[k];
    uint32_t r0 = 0, r1 = 0;
    uint32_t j = 0;
    for (; j + 2 <= lam; j += 2) {
      const ulonglong2 q = *reinterpret_cast<const ulonglong2*>(&keys[j]);
      r0 += q.x < kk;
      r1 += q.y < kk;
    }
    if (j < lam) r0 += keys[j] < kk;
    const uint32_t r = r0 + r1;
    if (r < top) out[r] = (int)k;
    if (r >= lam - top) out[top + (r - (lam - top))] = (int)k;
  }
}

// Block size of k_rank: 512 threads for short spark lists (C4, lambda = 30:
// 0.1254 -> 0.1244 ms per generation), 1024 otherwise (the counting rank
// needs a thread per spark and splits the range for lambda <= 512).
static unsigned rank_threads(const EngineView& v) { return v.lam <= 128 ? 512u : (unsigned)kRankThreads; }

static size_t rank_smem(const EngineView& v) {
  const size_t keys = ((v.lam + 1) & ~1ull) * sizeof(uint64_t);
  const bool split = v.lam * 2 <= (uint64_t)kRankThreads && v.lam * 12 <= (uint64_t)kRankSmemMax;
  return keys + (split ? v.lam * sizeof(uint32_t) : 0);
}

// ----------------------------------------------------------------- guides
// guiding_vector (engine.cpp:159-168, fp64, pairwise in rank order, then
// / top) + multi_guiding_sparks (pos + beta_m * delta, engine.cpp:189) +
// random_mapping(kGuide) + fp32 / bf16 stores.  Work item = (firework,
// 128-coordinate slice): one float4 per lane, the top-row loop unrolled by 4
// so each lane keeps 8 independent 16-byte loads in flight (the kernel is a
// gather-reduce over 2*top spark rows, HBM-bound).  The analytic fitness of
// the guides is computed afterwards by k_analytic_partials (same grouping as
// every other fitness, so cached fitness == re-evaluated fitness bit-wise).
#ifndef GUIDES_VEC
#define GUIDES_VEC 2  // coordinates per lane (2: float2, 4: float4; measured: 4 is slower on C2, 13.1 -> 15.2 us)
#endif
template <int V> struct VecT;
template <> struct VecT<2> { using T = float2; };
template <> struct VecT<4> { using T = float4; };
template <int V>
__device__ __forceinline__ void vec_split(const typename VecT<V>::T& q, float (&o)[V]) {
  if constexpr (V == 2) {
    o[0] = q.x, o[1] = q.y;
  } else {
    o[0] = q.x, o[1] = q.y, o[2] = q.z, o[3] = q.w;
  }
}

template <int V>
__device__ __forceinline__ void store_guide(const EngineView& v, uint64_t off, const float (&x)[V]) {
  if constexpr (V == 2) {
    *reinterpret_cast<float2*>(v.guides + off) = make_float2(x[0], x[1]);
    if (v.nn) *reinterpret_cast<__nv_bfloat162*>(v.guides_h + off) = __floats2bfloat162_rn(x[0], x[1]);
  } else {
    *reinterpret_cast<float4*>(v.guides + off) = make_float4(x[0], x[1], x[2], x[3]);
    if (v.nn) store_bf16x4(v.guides_h, off, x);
  }
}

#ifndef GUIDES_LDCS
#define GUIDES_LDCS 1  // the rank-row loads with the evict-first (streaming) hint (C2 0.2683 -> 0.2651 ms)
#endif
#if GUIDES_LDCS
#define GUIDE_LD(p) __ldcs(reinterpret_cast<const VT*>(p))
#else
#define GUIDE_LD(p) (*reinterpret_cast<const VT*>(p))
#endif
#ifndef GUIDES_WARPS
#define GUIDES_WARPS 8  // warps per k_guides block (one 32 * GUIDES_VEC-coordinate slice each)
#endif
constexpr int kGuideWarps = GUIDES_WARPS;
// U: rank pairs per unrolled load step (2U independent V-wide loads per
// lane in flight): 30 when top <= 64 (C2: top = 60 in two load rounds,
// 27.2 -> 25.7 us), else 16 (20 measured slower on both C2 and C5).
template <int U>
__global__ void __launch_bounds__(kGuideWarps * 32) k_guides(EngineView v) {
  constexpr int V = GUIDES_VEC;
  using VT = typename VecT<V>::T;
  pdl_enter();
  if (gen_inactive(v)) return;
  extern __shared__ uint64_t s_pre[];  // [M] kGuide key prefixes, then [2*top] rank lists
  int* s_idx = reinterpret_cast<int*>(s_pre + v.M);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t it = v.ctl->iteration;
  const uint64_t nsl = (v.D + 32 * V - 1) / (32 * V);  // 32V-coordinate slices (V per lane)
  const uint64_t bpf = (nsl + kGuideWarps - 1) / kGuideWarps;  // blocks per firework
  const uint64_t top = v.top;
  for (uint64_t blk = blockIdx.x; blk < v.Fl * bpf; blk += gridDim.x) {
    const uint64_t fl = blk / bpf, f = v.f_lo + fl;  // local / global firework
    const uint64_t c = (blk % bpf) * kGuideWarps + warp;
    const uint64_t b = f / v.mu, n = f % v.mu;
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < 2 * top; i += blockDim.x) s_idx[i] = v.rank_idx[fl * 2 * top + i];
    // hoisted rng.hpp:43-51 up to field m: one splitmix64 round per coordinate
    for (uint64_t m = threadIdx.x; m < v.M; m += blockDim.x) s_pre[m] = key_prefix(v.seed, kGuide, it, b, n, m);
    __syncthreads();
    const uint64_t d0 = c * 32 * V + lane * V;
    if (c >= nsl || d0 >= v.D) continue;
    const float* sb = v.sparks + fl * v.lam * v.Dp + d0;
    double acc[V];
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] = 0.0;
    uint64_t t = 0;
    // 2U independent loads in flight per lane, summed in rank order
    for (; t + U <= top; t += U) {
      VT bb[U], ww[U];
#pragma unroll
      for (int i = 0; i < U; ++i) {
        bb[i] = GUIDE_LD(sb + (uint64_t)s_idx[t + i] * v.Dp);
        ww[i] = GUIDE_LD(sb + (uint64_t)s_idx[top + t + i] * v.Dp);
      }
#pragma unroll
      for (int i = 0; i < U; ++i) {
        float bf_[V], wf_[V];
        vec_split<V>(bb[i], bf_);
        vec_split<V>(ww[i], wf_);
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] = __dadd_rn(acc[e], __dsub_rn((double)bf_[e], (double)wf_[e]));
      }
    }
    for (; t + 4 <= top; t += 4) {
      VT bb[4], ww[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        bb[i] = GUIDE_LD(sb + (uint64_t)s_idx[t + i] * v.Dp);
        ww[i] = GUIDE_LD(sb + (uint64_t)s_idx[top + t + i] * v.Dp);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float bf_[V], wf_[V];
        vec_split<V>(bb[i], bf_);
        vec_split<V>(ww[i], wf_);
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] = __dadd_rn(acc[e], __dsub_rn((double)bf_[e], (double)wf_[e]));
      }
    }
    for (; t < top; ++t) {
      float bf_[V], wf_[V];
      vec_split<V>(GUIDE_LD(sb + (uint64_t)s_idx[t] * v.Dp), bf_);
      vec_split<V>(GUIDE_LD(sb + (uint64_t)s_idx[top + t] * v.Dp), wf_);
#pragma unroll
      for (int e = 0; e < V; ++e) acc[e] = __dadd_rn(acc[e], __dsub_rn((double)bf_[e], (double)wf_[e]));
    }
    const double dtop = (double)top;
    double delta[V];
#pragma unroll
    for (int e = 0; e < V; ++e) delta[e] = __ddiv_rn(acc[e], dtop);
    float pv[V];
    vec_split<V>(*reinterpret_cast<const VT*>(v.pos + f * v.Dp + d0), pv);
    const float* plo = v.pop_lo + b * v.Dp;
    const float* phi = v.pop_hi + b * v.Dp;
    for (uint64_t m = 0; m < v.M; ++m) {
      const double beta = v.boosts[m];
      const uint64_t pg = s_pre[m];
      float x[V];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const uint64_t d = d0 + e;
        if (d < v.D) {
          const double gx = __dadd_rn((double)pv[e], __dmul_rn(beta, delta[e]));
          x[e] = map_coord(v, gx, d, pg, plo, phi);
        } else {
          x[e] = 0.0f;
        }
      }
      store_guide<V>(v, (fl * v.M + m) * v.Dp + d0, x);  // local guide row
    }
  }
}

// ----------------------------------------------------------------- select
// select_best (engine.cpp:198-242): strict-< scan firework -> sparks k up ->
// guides m up == lexicographic min of (value, scan order).  Then
// update_amplitudes (engine.cpp:244-256), the wave accounting
// (engine.cpp:388-390) and the winner row copy (engine.cpp:232-233).  One
// block per firework.
#ifndef SELECT_THREADS
#define SELECT_THREADS 512
#endif
constexpr int kSelectThreads = SELECT_THREADS;
// select_best + update_amplitudes + wave accounting + winner copy for local
// firework fl, given the guide fitness gs[M] (all threads of the block;
// any block size that is a multiple of 32, at most 1024).
__device__ void select_core(const EngineView& v, uint64_t fl, const float* gs, unsigned nan_local,
                            const double* old_fit, uint32_t part, uint32_t nparts);

// grid (Fl, parts): parts > 1 split the winner copy; they need k_rank's
// fit_prev (parts == 1 reads fit directly: the operator seam).
__global__ void __launch_bounds__(kSelectThreads) k_select(EngineView v) {
  pdl_enter<true>();
  if (gen_inactive(v)) return;
  const uint64_t fl = blockIdx.x;  // local firework
  const uint32_t part = blockIdx.y, nparts = gridDim.y;
  __shared__ float gs[16];
  unsigned nan_local = 0;
  // guide fitness: one warp per guide row (warp-cooperative finalize)
  for (uint64_t m = threadIdx.x >> 5; m < v.M; m += blockDim.x >> 5) {
    float g;
    if (v.injected_fitness) {
      g = v.gfit[fl * v.M + m];
    } else {
      bool nan;
      g = finalize_row(v, v.gpart, fl * v.M + m, &nan);
      nan_local += nan && (threadIdx.x & 31) == 0;  // once per row (select_core sums lanes)
      if ((threadIdx.x & 31) == 0 && part == 0) v.gfit[fl * v.M + m] = g;
    }
    if ((threadIdx.x & 31) == 0) gs[m] = g;
  }
  __syncthreads();
  select_core(v, fl, gs, nan_local, nparts > 1 ? v.fit_prev : v.fit, part, nparts);
}

// The decision is computed by every part (from old_fit, which part 0's state
// update does not touch); part 0 writes the state, part p copies slice p of
// the winner row.
__device__ void select_core(const EngineView& v, uint64_t fl, const float* gs, unsigned nan_local,
                            const double* old_fit, uint32_t part, uint32_t nparts) {
  const uint64_t f = v.f_lo + fl;  // global firework
  __shared__ double sv[32];
  __shared__ int so[32];
  __shared__ int s_win;
  double best_v = old_fit[f];
  int best_o = 0;
  if (threadIdx.x != 0) best_v = __longlong_as_double(0x7ff0000000000000ll), best_o = 0x7fffffff;
  for (uint64_t k = threadIdx.x; k < v.lam; k += blockDim.x) {
    const double x = (double)v.sfit[fl * v.lam + k];
    const int o = 1 + (int)k;
    if (x < best_v || (x == best_v && o < best_o)) best_v = x, best_o = o;
  }
  for (uint64_t m = threadIdx.x; m < v.M; m += blockDim.x) {
    const double x = (double)gs[m];
    const int o = 1 + (int)v.lam + (int)m;
    if (x < best_v || (x == best_v && o < best_o)) best_v = x, best_o = o;
  }
  // warp then block lexicographic min
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best_v, off);
    const int oo = __shfl_xor_sync(0xffffffffu, best_o, off);
    if (ov < best_v || (ov == best_v && oo < best_o)) best_v = ov, best_o = oo;
  }
  nan_local = __reduce_add_sync(0xffffffffu, nan_local);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sv[w] = best_v;
    so[w] = best_o;
    if (nan_local && part == 0) atomicAdd(nan_counter_own(v), (unsigned long long)nan_local);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
      if (sv[i] < best_v || (sv[i] == best_v && so[i] < best_o)) best_v = sv[i], best_o = so[i];
    // If every candidate is NaN-free but the firework is +inf and all are
    // +inf, the firework (order 0) wins: strict < never fires.
    const double old = old_fit[f];
    if (!(best_v < old)) {
      best_v = old;
      best_o = 0;
    }
    s_win = best_o;
    if (part == 0) {
      const double gain = old - best_v;
      v.fit[f] = best_v;
      v.li[f] = (0.0 < gain) ? gain : 0.0;
      const int imp = best_v < old;
      v.improved[f] = imp;
      v.winner[f] = best_o;
      const double a = v.amp[f] * (imp ? v.amp_amplify : v.amp_reduce);
      v.amp[f] = a < v.amp_floor ? v.amp_floor : (v.max_range < a ? v.max_range : a);
      if (fl == 0) v.ctl->used += v.wave;  // the global wave, on every rank
    }
  }
  __syncthreads();
  // winner row -> firework row (padding included: rows are Dp wide)
  const int win = s_win;
  if (win == 0) return;
  const float4* src = reinterpret_cast<const float4*>(
      (uint64_t)win <= v.lam ? v.sparks + (fl * v.lam + (win - 1)) * v.Dp
                             : v.guides + (fl * v.M + (win - 1 - v.lam)) * v.Dp);
  float4* dst = reinterpret_cast<float4*>(v.pos + f * v.Dp);
  const uint64_t n4all = (v.D + 3) / 4;
  const uint64_t q0 = n4all * part / nparts, q1 = n4all * (part + 1) / nparts;
  src += q0;
  dst += q0;
  const uint64_t n4 = q1 - q0;
  const uint32_t nt = blockDim.x;
  uint64_t i = threadIdx.x;
  for (; i + 3 * nt < n4; i += 4 * nt) {
    float4 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = src[i + u * nt];
#pragma unroll
    for (int u = 0; u < 4; ++u) dst[i + u * nt] = t[u];
  }
  for (; i < n4; i += nt) dst[i] = src[i];
}

// ------------------------------------------------------------------ loser
// iterations_remaining of the current generation, engine.cpp:394-410.
__device__ double iters_remaining(const EngineView& v) {
  double iters_rem = 0.0;
  if (v.has_iters_override) {
    iters_rem = v.iters_override;
  } else if (v.max_evals > 0) {
    const uint64_t used = v.ctl->used;
    const uint64_t left = v.max_evals > used ? v.max_evals - used : 0;
    iters_rem = (double)left / (double)v.wave;
  } else {
    const double now_ms = (double)(global_ns() - v.ctl->start_ns) * 1e-6;
    const double avg = (now_ms - v.ctl->init_ms) / (double)v.ctl->iteration;
    if (avg > 0.0) {
      const double rem = v.wall_budget_ms - now_ms;
      iters_rem = (rem > 0.0 ? rem : 0.0) / avg;
    }
  }
  return iters_rem;
}

// loser_out decision (engine.cpp:258-286) with iterations_remaining from
// engine.cpp:394-410 (device clock for the wall-clock budget).  One block.
__global__ void k_loser(EngineView v) {
  pdl_enter<true>();
  __shared__ int count;
  if (threadIdx.x == 0) count = 0;
  __syncthreads();
  if (gen_inactive(v)) {
    if (threadIdx.x == 0) v.ctl->n_losers = 0, v.ctl->n_losers_all = 0;
    return;
  }
  const double iters_rem = iters_remaining(v);
  for (uint64_t b = v.b_lo + threadIdx.x; b < v.b_hi; b += blockDim.x) {
    // argmin_per_population (backend.cpp:69-83)
    uint64_t bi = 0;
    double bv = v.fit[b * v.mu];
    for (uint64_t n = 1; n < v.mu; ++n)
      if (v.fit[b * v.mu + n] < bv) bv = v.fit[b * v.mu + n], bi = n;
    int cnt = 0;
    for (uint64_t n = 0; n < v.mu; ++n) {
      const uint64_t f = b * v.mu + n;
      int is_loser = 0;
      if (iters_rem > 0.0 && n != bi) {
        // projected = f - li * iters_rem, rounded like the reference (no FMA)
        const double projected = __dsub_rn(v.fit[f], __dmul_rn(v.li[f], iters_rem));
        is_loser = projected > bv;
      }
      v.loser[f] = is_loser;
      if (is_loser) {
        v.amp[f] = v.a0;
        v.li[f] = 0.0;
        ++cnt;
      }
    }
    atomicAdd(&count, cnt);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    v.ctl->iters_rem = iters_rem;
    v.ctl->n_losers = count;
    if (v.replica) {
      v.ctl->n_losers_all = (uint64_t)count;  // the exchange adds the other shards' counts
    } else {
      v.ctl->used += (uint64_t)count;
      v.ctl->losers_total += (uint64_t)count;
    }
  }
}

// Replica sharding, in-process exchange (tests): add another shard's loser
// count of this generation.
__global__ void k_fold_nan(Ctl* ctl) {
  ctl->nan_count += ctl->nan_all;
  ctl->nan_own = ctl->nan_all = 0;
}
void launch_fold_nan(Ctl* ctl, cudaStream_t s) { k_fold_nan<<<1, 1, 0, s>>>(ctl); }

__global__ void k_add_losers(Ctl* dst, const Ctl* src, int losers) {
  if (losers) dst->n_losers_all += (uint64_t)src->n_losers;
  dst->nan_all += src->nan_own;
}

// ------------------------------------------------------------ fresh rows
// mode 0: initialize (engine.cpp:56-64): every firework, kInit, iteration 0.
// mode 1: loser reinit (engine.cpp:287-294): losers only, kReinit.
__global__ void __launch_bounds__(256) k_fresh_rows(EngineView v, int mode) {
  pdl_enter<true>();
  if (mode == 1 && (gen_inactive(v) || v.ctl->n_losers == 0)) return;
  if (mode == 0 && blockIdx.x == 0 && threadIdx.x == 0) v.ctl->start_ns = global_ns();
  const int lane = threadIdx.x & 31;
  const uint64_t it = mode == 0 ? 0 : v.ctl->iteration;
  const uint64_t stream = mode == 0 ? kInit : kReinit;
  const uint64_t items = v.F * v.nch;
  for (uint64_t item = blockIdx.x * (uint64_t)kWarps + (threadIdx.x >> 5);
       item < items; item += (uint64_t)gridDim.x * kWarps) {
    const uint64_t f = item / v.nch, c = item % v.nch;
    if (mode == 1 && (!v.loser[f] || f < v.b_lo * v.mu || f >= v.b_hi * v.mu)) continue;
    const uint64_t b = f / v.mu, n = f % v.mu;
    const uint64_t pk = key_prefix(v.seed, stream, it, b, n, 0);
    float s0 = 0.0f, s1 = 0.0f;
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {
      const uint64_t d0 = c * kChunk + q * 128 + lane * 4;
      if (d0 >= v.D) break;
      float x[4];
      float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint64_t d = d0 + e;
        if (d < v.D) {
          const double u = uniform_draw(splitmix64(pk ^ d), v.lower[d], v.upper[d]);
          x[e] = to_f32_in_box(u, v.lower_f[d], v.upper_f[d]);
          if (!v.nn) analytic_terms(v.obj_kind, x[e], a0, a1);
        } else {
          x[e] = 0.0f;
        }
      }
      s0 += a0;
      s1 += a1;
      *reinterpret_cast<float4*>(v.pos + f * v.Dp + d0) = make_float4(x[0], x[1], x[2], x[3]);
      if (v.nn) store_bf16x4(v.fresh_h, f * v.Dp + d0, x);
    }
    if (!v.nn) {
      s0 = warp_sum(s0);
      s1 = warp_sum(s1);
      if (lane == 0) {
        v.fpart[(f * v.nparts + c) * 2] = s0;
        v.fpart[(f * v.nparts + c) * 2 + 1] = s1;
      }
    }
  }
}

// ------------------------------------------------------- finalize/record
// mode 0 (end of initialize, engine.cpp:66-74 + record_wave #0) or mode 1
// (loser fitness commit engine.cpp:298-309 + record_wave engine.cpp:416).
// record_wave (engine.cpp:340-351): per-batch argmin; best only on strict
// improvement; one trace point per batch.  Then the loop-top termination
// test (engine.cpp:360-367) for the next generation.  One block.
__global__ void k_finalize_record(EngineView v, int mode) {
  pdl_enter<true>();
  Ctl* ctl = v.ctl;
  if (mode == 1 && v.nan_mode) {
    // fold the shards' NaN counts of this generation's exchange (Ctl::nan_own)
    if (threadIdx.x == 0) {
      ctl->nan_count += v.nan_mode == 2 ? ctl->nan_all : ctl->nan_own + ctl->nan_all;
      ctl->nan_own = ctl->nan_all = 0;
    }
    __syncthreads();
  }
  if (mode == 1 && gen_inactive(v)) {
    for (uint64_t b = threadIdx.x; b < v.B; b += blockDim.x) v.rec_flag[b] = 0;
    return;
  }
  unsigned nan_local = 0;
  const int lane = threadIdx.x & 31;
  for (uint64_t f = threadIdx.x >> 5; f < v.F; f += blockDim.x >> 5) {  // one warp per row
    if (mode == 0 || (v.loser[f] && f >= v.b_lo * v.mu && f < v.b_hi * v.mu)) {
      bool nan;
      const float x = finalize_row(v, v.fpart, f, &nan);
      nan_local += nan;
      if (lane == 0) {
        v.fit[f] = (double)x;
        if (mode == 0) {
          v.amp[f] = v.a0;
          v.li[f] = 0.0;
        }
      }
    }
  }
  // replica shards evaluate only their own batches' losers: shard-local work
  if (lane == 0 && nan_local)
    atomicAdd(mode == 1 && v.replica ? nan_counter_own(v) : (unsigned long long*)&ctl->nan_count,
              (unsigned long long)nan_local);
  __syncthreads();
  if (mode == 0 && threadIdx.x == 0) {
    ctl->used = v.F;
    ctl->losers_total = 0;
    ctl->trace_n = 0;
    ctl->gens_run = 0;
  }
  if (mode == 1 && v.replica && threadIdx.x == 0) {  // losers of every shard (exchanged)
    ctl->used += ctl->n_losers_all;
    ctl->losers_total += ctl->n_losers_all;
  }
  __syncthreads();
  const uint64_t now = global_ns();
  const uint64_t slot = ctl->trace_n % v.trace_cap;
  for (uint64_t b = threadIdx.x; b < v.B; b += blockDim.x) {
    if (mode == 1 && (b < v.b_lo || b >= v.b_hi)) {  // another shard's batch: not tracked here
      v.rec_flag[b] = 0;
      v.tr_evals[slot * v.B + b] = ctl->used;
      v.tr_best[slot * v.B + b] = __longlong_as_double(0x7ff8000000000000ll);
      v.tr_ns[slot * v.B + b] = now - ctl->start_ns;
      continue;
    }
    uint64_t bi = 0;
    double bv = v.fit[b * v.mu];
    for (uint64_t n = 1; n < v.mu; ++n)
      if (v.fit[b * v.mu + n] < bv) bv = v.fit[b * v.mu + n], bi = n;
    double cur = mode == 0 ? __longlong_as_double(0x7ff0000000000000ll) : v.best_fit[b];
    int flag = 0;
    if (bv < cur) {
      cur = bv;
      v.best_idx[b] = (int)bi;
      flag = 1;
    }
    v.best_fit[b] = cur;
    v.rec_flag[b] = flag;
    v.tr_evals[slot * v.B + b] = ctl->used;
    v.tr_best[slot * v.B + b] = cur;
    v.tr_ns[slot * v.B + b] = now - ctl->start_ns;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ctl->trace_n += 1;
    const double now_ms = (double)(now - ctl->start_ns) * 1e-6;
    if (mode == 0) {
      ctl->init_ms = now_ms;
      ctl->iteration = 0;
    } else {
      ctl->gens_run += 1;
    }
    int active = 1;
    if (v.max_evals > 0 && ctl->used >= v.max_evals) active = 0;
    if (v.wall_budget_ms > 0.0 && now_ms >= v.wall_budget_ms) active = 0;
    ctl->active = active;
    if (active) ctl->iteration += 1;
  }
}

// Tail of a generation (and of initialize): the best-position copy on strict
// improvement (engine.cpp:343-346) and population_range (engine.cpp:22-41)
// of the NEXT generation's pre-selection state, which is final here.  One
// float4 of coordinates per thread (grid-stride), the mu rows' loads in
// flight together.
__global__ void __launch_bounds__(256) k_record_copy(EngineView v) {
  pdl_enter<true>();
  const uint64_t n4 = (v.D + 3) / 4, items = (v.b_hi - v.b_lo) * n4;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < items;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = v.b_lo + i / n4, d0 = (i % n4) * 4;
    const float* pb = v.pos + b * v.mu * v.Dp + d0;
    if (v.rec_flag[b])
      *reinterpret_cast<float4*>(v.best_pos + b * v.Dp + d0) =
          *reinterpret_cast<const float4*>(pb + (uint64_t)v.best_idx[b] * v.Dp);
    // std::min / std::max keep-first order over n = 0..mu-1
    float4 mn = *reinterpret_cast<const float4*>(pb), mx = mn;
    uint64_t n = 1;
    for (; n + 4 <= v.mu; n += 4) {
      float4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = *reinterpret_cast<const float4*>(pb + (n + u) * v.Dp);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        mn.x = x[u].x < mn.x ? x[u].x : mn.x;
        mn.y = x[u].y < mn.y ? x[u].y : mn.y;
        mn.z = x[u].z < mn.z ? x[u].z : mn.z;
        mn.w = x[u].w < mn.w ? x[u].w : mn.w;
        mx.x = mx.x < x[u].x ? x[u].x : mx.x;
        mx.y = mx.y < x[u].y ? x[u].y : mx.y;
        mx.z = mx.z < x[u].z ? x[u].z : mx.z;
        mx.w = mx.w < x[u].w ? x[u].w : mx.w;
      }
    }
    for (; n < v.mu; ++n) {
      const float4 x = *reinterpret_cast<const float4*>(pb + n * v.Dp);
      mn.x = x.x < mn.x ? x.x : mn.x;
      mn.y = x.y < mn.y ? x.y : mn.y;
      mn.z = x.z < mn.z ? x.z : mn.z;
      mn.w = x.w < mn.w ? x.w : mn.w;
      mx.x = mx.x < x.x ? x.x : mx.x;
      mx.y = mx.y < x.y ? x.y : mx.y;
      mx.z = mx.z < x.z ? x.z : mx.z;
      mx.w = mx.w < x.w ? x.w : mx.w;
    }
    *reinterpret_cast<float4*>(v.pop_lo + b * v.Dp + d0) = mn;
    *reinterpret_cast<float4*>(v.pop_hi + b * v.Dp + d0) = mx;
  }
}

static unsigned tail_blocks(const EngineView& v, int nsm) {
  const uint64_t g = (v.B * ((v.D + 3) / 4) + 255) / 256;
  const uint64_t cap = (uint64_t)nsm * 8;
  return (unsigned)(g == 0 ? 1 : (g < cap ? g : cap));
}

// ------------------------------------------------------ small problems
// One context, analytic objective, D <= kChunk: the post-explode part of a
// generation as two kernels instead of eight (the launch latency dominates
// at these sizes, e.g. C1: D = 30, 165 evaluations per generation).  Every
// value is computed with the same operation order as the general kernels
// (tests compare the two paths bit for bit through the sharded runs).
//
// k_small_a, one block per firework: spark-fitness finalize + ranking
// (k_rank), guiding vector + guides + kGuide mapping (k_guides), guide
// fitness (k_analytic_partials + the finalize of k_select), selection,
// amplitudes, wave accounting and winner copy (k_select); block 0 also
// fixes iterations_remaining for the loser decision (k_loser's value).
constexpr int kSmallThreads = 256;

// Analytic partial sums of one <= kChunk row, exactly as k_analytic_partials
// (per-4 groups, lane-strided, warp butterfly), finalized as finalize_rows
// (lane 0's value).  Whole warp.
__device__ __forceinline__ float small_row_fitness(const EngineView& v, const float* row,
                                                   float* part, bool* was_nan) {
  const int lane = threadIdx.x & 31;
  float s0 = 0.0f, s1 = 0.0f;
  for (int q = 0; q < 4; ++q) {
    const uint64_t d0 = q * 128 + lane * 4;
    if (d0 >= v.D) break;
    const float4 x4 = *reinterpret_cast<const float4*>(row + d0);
    const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
    float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (d0 + e < v.D) analytic_terms(v.obj_kind, xs[e], a0, a1);
    s0 += a0;
    s1 += a1;
  }
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  if (lane == 0 && part != nullptr) {
    part[0] = s0;
    part[1] = s1;
  }
  // finalize_rows with nparts == 1: the partial itself (0 + p0, row_sums_seq)
  const float a = __shfl_sync(0xffffffffu, warp_sum(lane == 0 ? s0 : 0.0f), 0);
  const float b = __shfl_sync(0xffffffffu, warp_sum(lane == 0 ? s1 : 0.0f), 0);
  const float f = analytic_finalize(v.obj_kind, a, b, v.D);
  *was_nan = isnan(f);
  return isnan(f) ? __int_as_float(0x7f800000) : f;
}

// Phase A of local firework fl (all threads of the block; sa_keys: lam
// uint64 of shared memory).
__device__ void small_a_body(const EngineView& v, uint64_t fl, uint64_t* sa_keys) {
  __shared__ int s_idx[2 * 1024];        // top / bottom spark indices (top <= 1024)
  __shared__ float gs[16];
  const uint64_t f = v.f_lo + fl;
  const uint32_t lam = (uint32_t)v.lam, top = (uint32_t)v.top;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const uint64_t it = v.ctl->iteration;
  unsigned nan_local = 0;
  // ---- spark fitness (finalize) + keys
  constexpr int R = 4;
  for (uint32_t k0 = warp * R; k0 < lam; k0 += nwarp * R) {
    int64_t rows[R];
    float x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rows[r] = (k0 + r < lam) ? (int64_t)(fl * lam + k0 + r) : -1;
    unsigned nan_rows = 0;  // equal on every lane: counted once (select_core sums the warp)
    finalize_rows<R>(v, v.spart, rows, x, nan_rows);
    nan_local += lane == 0 ? nan_rows : 0u;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (lane == r && rows[r] >= 0) {
        v.sfit[rows[r]] = x[r];
        sa_keys[k0 + r] = rank_key(x[r], k0 + r);
      }
  }
  __syncthreads();
  if (v.M > 0) {
    // ---- counting rank (k_rank)
    for (uint32_t k = threadIdx.x; k < lam; k += blockDim.x) {
      const uint64_t kk = sa_keys[k];
      uint32_t r = 0;
      for (uint32_t j = 0; j < lam; ++j) r += sa_keys[j] < kk;
      if (r < top) s_idx[r] = (int)k;
      if (r >= lam - top) s_idx[top + (r - (lam - top))] = (int)k;
    }
    __syncthreads();
    // ---- guiding vector + guides + kGuide mapping (k_guides)
    const uint64_t b = f / v.mu, n = f % v.mu;
    const float* sb = v.sparks + fl * v.lam * v.Dp;
    const float* plo = v.pop_lo + b * v.Dp;
    const float* phi = v.pop_hi + b * v.Dp;
    const uint64_t d4 = (v.D + 3) & ~3ull;
    __shared__ uint64_t s_gpre[16];  // kGuide key prefixes (M <= 16)
    for (uint64_t m = threadIdx.x; m < v.M; m += blockDim.x) s_gpre[m] = key_prefix(v.seed, kGuide, it, b, n, m);
    __syncthreads();
    for (uint64_t d = threadIdx.x; d < d4; d += blockDim.x) {
      if (d >= v.D) {
        for (uint64_t m = 0; m < v.M; ++m) v.guides[(fl * v.M + m) * v.Dp + d] = 0.0f;
        continue;
      }
      double acc = 0.0;
      uint32_t t = 0;
      // rank pairs 8 at a time, all 16 loads in flight, summed in rank order
      for (; t + 8 <= top; t += 8) {
        float tv[8], bv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          tv[i] = sb[(uint64_t)s_idx[t + i] * v.Dp + d];
          bv[i] = sb[(uint64_t)s_idx[top + t + i] * v.Dp + d];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) acc = __dadd_rn(acc, __dsub_rn((double)tv[i], (double)bv[i]));
      }
      if (t < top) {
        float tv[8], bv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t ti = t + i < top ? t + i : t;
          tv[i] = sb[(uint64_t)s_idx[ti] * v.Dp + d];
          bv[i] = sb[(uint64_t)s_idx[top + ti] * v.Dp + d];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (t + i < top) acc = __dadd_rn(acc, __dsub_rn((double)tv[i], (double)bv[i]));
      }
      const double delta = __ddiv_rn(acc, (double)top);
      const double pv = (double)v.pos[f * v.Dp + d];
      for (uint64_t m = 0; m < v.M; ++m) {
        const uint64_t pg = s_gpre[m];
        const double gx = __dadd_rn(pv, __dmul_rn(v.boosts[m], delta));
        v.guides[(fl * v.M + m) * v.Dp + d] = map_coord(v, gx, d, pg, plo, phi);
      }
    }
    __syncthreads();
    // ---- guide fitness, one warp per guide
    for (uint64_t m = warp; m < v.M; m += nwarp) {
      bool nan;
      const uint64_t row = fl * v.M + m;
      const float g = small_row_fitness(v, v.guides + row * v.Dp, v.gpart + row * 2, &nan);
      nan_local += nan && lane == 0;
      if (lane == 0) {
        v.gfit[row] = g;
        gs[m] = g;
      }
    }
    __syncthreads();
  }
  select_core(v, fl, gs, nan_local, v.fit, 0, 1);
  if (fl == 0 && threadIdx.x == 0) v.ctl->iters_rem = iters_remaining(v);  // after the wave
  __syncthreads();  // shared state (s_idx, gs, keys) free for the next firework
}

__global__ void __launch_bounds__(kSmallThreads) k_small_a(EngineView v) {
  pdl_enter<true>();
  if (gen_inactive(v)) return;
  extern __shared__ uint64_t sa_keys[];  // [lam] rank keys
  small_a_body(v, blockIdx.x, sa_keys);
}

// k_small_b, one block per batch: loser-out (k_loser), reinit + fitness of
// the losers (k_fresh_rows + k_finalize_record), record_wave, best copy and
// population_range of the next generation (k_record_copy); the last block
// to finish completes the trace point and the loop-top termination test.
// Phase B of batch b (all threads of the block); the last of the `nblocks`
// callers of a generation completes the trace point and the termination test.
__device__ void small_b_body(const EngineView& v, uint64_t b, unsigned nblocks) {
  Ctl* ctl = v.ctl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const uint64_t it = ctl->iteration;
  const uint64_t slot = ctl->trace_n % v.trace_cap;
  __shared__ int s_count;
  unsigned nan_local = 0;
  // loaded up front: record_wave needs them after the loser phase
  const double best_prev = threadIdx.x == 0 ? v.best_fit[b] : 0.0;
  const uint64_t start_ns = threadIdx.x == 0 ? ctl->start_ns : 0;
  // ---- loser decision for batch b (k_loser, engine.cpp:258-286)
  if (v.mu <= 32) {
    // warp 0, lane n = firework n: batch argmin as the lexicographic min of
    // (fitness, n) (== the strict-< scan), loser flags in parallel
    if (warp == 0) {
      const double iters_rem = ctl->iters_rem;
      const uint64_t f = b * v.mu + lane;
      const bool in = (uint64_t)lane < v.mu;
      const double fv = in ? v.fit[f] : __longlong_as_double(0x7ff0000000000000ll);
      const double lv = in ? v.li[f] : 0.0;
      double bv = fv;
      int bi = in ? lane : 0x7fffffff;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ov < bv || (ov == bv && oi < bi)) bv = ov, bi = oi;
      }
      int is_loser = 0;
      if (in && iters_rem > 0.0 && lane != bi) is_loser = __dsub_rn(fv, __dmul_rn(lv, iters_rem)) > bv;
      if (in) {
        v.loser[f] = is_loser;
        if (is_loser) {
          v.amp[f] = v.a0;
          v.li[f] = 0.0;
        }
      }
      const int cnt = __popc(__ballot_sync(0xffffffffu, is_loser));
      if (lane == 0) {
        s_count = cnt;
        if (cnt) {
          atomicAdd((unsigned long long*)&ctl->used, (unsigned long long)cnt);
          atomicAdd((unsigned long long*)&ctl->losers_total, (unsigned long long)cnt);
        }
      }
    }
  } else if (threadIdx.x == 0) {

    const double iters_rem = ctl->iters_rem;
    uint64_t bi = 0;
    double bv = v.fit[b * v.mu];
    for (uint64_t n = 1; n < v.mu; ++n)
      if (v.fit[b * v.mu + n] < bv) bv = v.fit[b * v.mu + n], bi = n;
    int cnt = 0;
    for (uint64_t n = 0; n < v.mu; ++n) {
      const uint64_t f = b * v.mu + n;
      int is_loser = 0;
      if (iters_rem > 0.0 && n != bi)
        is_loser = __dsub_rn(v.fit[f], __dmul_rn(v.li[f], iters_rem)) > bv;
      v.loser[f] = is_loser;
      if (is_loser) {
        v.amp[f] = v.a0;
        v.li[f] = 0.0;
        ++cnt;
      }
    }
    s_count = cnt;
    if (cnt) {
      atomicAdd((unsigned long long*)&ctl->used, (unsigned long long)cnt);
      atomicAdd((unsigned long long*)&ctl->losers_total, (unsigned long long)cnt);
    }
  }
  __syncthreads();
  // ---- losers: kReinit rows + fitness (k_fresh_rows mode 1, k_finalize_record)
  if (s_count) {
    for (uint64_t n = warp; n < v.mu; n += nwarp) {
      const uint64_t f = b * v.mu + n;
      if (!v.loser[f]) continue;
      const uint64_t pk = key_prefix(v.seed, kReinit, it, b, n, 0);
      for (int q = 0; q < 4; ++q) {
        const uint64_t d0 = q * 128 + lane * 4;
        if (d0 >= v.D) break;
        float x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint64_t d = d0 + e;
          x[e] = d < v.D ? to_f32_in_box(uniform_draw(splitmix64(pk ^ d), v.lower[d], v.upper[d]),
                                         v.lower_f[d], v.upper_f[d])
                         : 0.0f;
        }
        *reinterpret_cast<float4*>(v.pos + f * v.Dp + d0) = make_float4(x[0], x[1], x[2], x[3]);
      }
      __syncwarp();
      bool nan;
      const float x = small_row_fitness(v, v.pos + f * v.Dp, v.fpart + f * v.nparts * 2, &nan);
      nan_local += nan && lane == 0;
      if (lane == 0) v.fit[f] = (double)x;
    }
    if (lane == 0 && nan_local)
      atomicAdd((unsigned long long*)&ctl->nan_count, (unsigned long long)nan_local);
    __syncthreads();
  }
  // ---- record_wave for batch b (engine.cpp:340-351)
  __shared__ int s_flag, s_best;
  __shared__ double s_bv;
  __shared__ int s_bi;
  const uint64_t now = global_ns();
  if (v.mu <= 32 && warp == 0) {  // batch argmin (lowest index on ties), warp-parallel
    const bool in = (uint64_t)lane < v.mu;
    double bv = in ? v.fit[b * v.mu + lane] : __longlong_as_double(0x7ff0000000000000ll);
    int bi = in ? lane : 0x7fffffff;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov < bv || (ov == bv && oi < bi)) bv = ov, bi = oi;
    }
    if (lane == 0) s_bv = bv, s_bi = bi;
    __syncwarp();
  }
  if (threadIdx.x == 0) {
    uint64_t bi = 0;
    double bv;
    if (v.mu <= 32) {
      bv = s_bv;
      bi = (uint64_t)s_bi;
    } else {
      bv = v.fit[b * v.mu];
      for (uint64_t n = 1; n < v.mu; ++n)
        if (v.fit[b * v.mu + n] < bv) bv = v.fit[b * v.mu + n], bi = n;
    }
    double cur = best_prev;
    int flag = 0;
    if (bv < cur) {
      cur = bv;
      v.best_idx[b] = (int)bi;
      flag = 1;
    }
    v.best_fit[b] = cur;
    v.rec_flag[b] = flag;
    v.tr_best[slot * v.B + b] = cur;
    v.tr_ns[slot * v.B + b] = now - start_ns;
    s_flag = flag;
    s_best = (int)bi;
  }
  __syncthreads();
  // ---- best copy + population_range (k_record_copy)
  const float* pb = v.pos + b * v.mu * v.Dp;
  const uint64_t d4 = (v.D + 3) & ~3ull;
  for (uint64_t d = threadIdx.x; d < d4; d += blockDim.x) {
    if (s_flag) v.best_pos[b * v.Dp + d] = pb[(uint64_t)s_best * v.Dp + d];
    float mn = pb[d], mx = mn;
    for (uint64_t n = 1; n < v.mu; ++n) {
      const float x = pb[n * v.Dp + d];
      mn = x < mn ? x : mn;
      mx = mx < x ? x : mx;
    }
    v.pop_lo[b * v.Dp + d] = mn;
    v.pop_hi[b * v.Dp + d] = mx;
  }
  // ---- the last block: trace evaluations, termination (k_finalize_record);
  // a single batch block (nblocks == 1) is the last one by construction
  if (threadIdx.x == 0) {
    bool last = true;
    if (nblocks > 1) {
      __threadfence();
      const unsigned done = atomicAdd(&ctl->small_done, 1u);
      last = done == nblocks - 1;
      if (last) __threadfence();
    }
    if (last) {
      const uint64_t used = *(volatile uint64_t*)&ctl->used;
      for (uint64_t bb = 0; bb < v.B; ++bb) v.tr_evals[slot * v.B + bb] = used;
      if (nblocks > 1) ctl->small_done = 0;
      ctl->trace_n += 1;
      ctl->gens_run += 1;
      const double now_ms = (double)(now - start_ns) * 1e-6;
      int active = 1;
      if (v.max_evals > 0 && used >= v.max_evals) active = 0;
      if (v.wall_budget_ms > 0.0 && now_ms >= v.wall_budget_ms) active = 0;
      ctl->active = active;
      if (active) ctl->iteration += 1;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSmallThreads) k_small_b(EngineView v) {
  pdl_enter<true>();
  if (gen_inactive(v)) {
    if (threadIdx.x == 0) v.rec_flag[blockIdx.x] = 0;
    return;
  }
  small_b_body(v, blockIdx.x, gridDim.x);
}

// Grid-wide barrier of a cooperative launch (all blocks co-resident).
__device__ void grid_barrier(Ctl* ctl, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = &ctl->bar_gen;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(&ctl->bar_count, 1u) == nblocks - 1) {
      ctl->bar_count = 0;
      __threadfence();
      *gen = g + 1;
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// The whole generation loop of a small problem in one persistent launch:
// one block per firework, up to max_gens generations: explode + mapping +
// fitness and phase A of the block's firework, a grid barrier
// (iterations_remaining after the global wave), phase B of the batch by its
// first firework's block, a grid barrier (termination test).  No launch
// latency between phases; every value is computed with the same device
// functions, in the same order, as the multi-kernel path.
// All the blocks form one thread-block cluster (F <= 8): the hardware cluster
// barrier (release / acquire at cluster scope) instead of the global-atomic
// grid barrier.
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Candidate buffers of the cluster form (SM = true): the block's sparks,
// guides, their partial sums and fitness live in shared memory for the whole
// launch (the EngineView the phase functions see is rebased onto them; the
// indexing by the global firework is unchanged) and are written through to
// HBM once per generation for the host-side readers (mgfwa_get_candidates).
struct SmallSmem {
  uint64_t sp, spart, gd, gpart, sfit, gfit, total;  // byte offsets after the keys
};
__host__ __device__ inline SmallSmem small_smem_layout(const EngineView& v) {
  SmallSmem L;
  uint64_t o = 0;
  auto take = [&](uint64_t bytes) { const uint64_t r = o; o += (bytes + 15) & ~15ull; return r; };
  L.sp = take(v.lam * v.Dp * 4);
  L.spart = take(v.lam * v.nparts * 2 * 4);
  L.gd = take(v.M * v.Dp * 4);
  L.gpart = take(v.M * 2 * 4);
  L.sfit = take(v.lam * 4);
  L.gfit = take(v.M * 4);
  L.total = o;
  return L;
}
template <typename T>
__device__ __forceinline__ T* rebase(uint8_t* base, uint64_t off, uint64_t elems_before) {
  return reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(base + off) - elems_before * sizeof(T));
}
__device__ __forceinline__ void copy_words(float* dst, const float* src, uint64_t n) {
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// Block size and explode spark-group size of the small-problem loop (256 / 4
// measured best on C1: 512 / 1 18.6, 256 / 2 17.3, 1024 / 1 20.9 vs 17.0 us).
#ifndef SMALL_RUN_KG
#define SMALL_RUN_KG 4
#endif
#ifndef SMALL_RUN_THREADS
#define SMALL_RUN_THREADS 256
#endif
constexpr int kSmallRunThreads = SMALL_RUN_THREADS;
constexpr int kSmallRunWarps = kSmallRunThreads / 32;

template <int KIND, bool CL, bool SM>
__global__ void __launch_bounds__(kSmallRunThreads) k_small_run(EngineView v, uint64_t max_gens) {
  extern __shared__ __align__(16) uint8_t run_smem[];
  ExplodeChunk& ch = *reinterpret_cast<ExplodeChunk*>(run_smem);
  ExplodeWarp* wqs = reinterpret_cast<ExplodeWarp*>(run_smem + sizeof(ExplodeChunk));
  uint64_t* keys =
      reinterpret_cast<uint64_t*>(run_smem + sizeof(ExplodeChunk) + kSmallRunWarps * sizeof(ExplodeWarp));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t f = blockIdx.x, b = f / v.mu;
  EngineView w = v;  // SM: the phases' view of this block's candidates
  if (SM) {
    uint8_t* cb = reinterpret_cast<uint8_t*>(keys + ((v.lam + 1) & ~1ull));
    const SmallSmem L = small_smem_layout(v);
    w.sparks = rebase<float>(cb, L.sp, f * v.lam * v.Dp);
    w.spart = rebase<float>(cb, L.spart, f * v.lam * v.nparts * 2);
    w.guides = rebase<float>(cb, L.gd, f * v.M * v.Dp);
    w.gpart = rebase<float>(cb, L.gpart, f * v.M * 2);
    w.sfit = rebase<float>(cb, L.sfit, f * v.lam);
    w.gfit = rebase<float>(cb, L.gfit, f * v.M);
  }
  for (uint64_t gen = 0; gen < max_gens; ++gen) {
    if (*(volatile int*)&v.ctl->active == 0) break;  // uniform: set before the last barrier
    // explode + mapping + fused fitness partials of firework f (one chunk: D <= kChunk)
    stage_explode_chunk(v, ch, b, 0);
    __syncthreads();
    const ulonglong2 hs = explode_stream_prefixes(v);
    constexpr int KGS = SMALL_RUN_KG;  // sparks per warp group
    for (uint64_t g = warp; g * KGS < v.lam; g += kSmallRunWarps)
      explode_group<KIND, KGS>(w, ch, wqs[warp], lane, 0, f, g, hs);
    __syncthreads();
    small_a_body(w, f, keys);
    if (CL) cluster_barrier(); else grid_barrier(v.ctl, gridDim.x);  // iterations_remaining (block 0) is final
    if (f % v.mu == 0) small_b_body(v, b, (unsigned)v.B);
    if (CL) cluster_barrier(); else grid_barrier(v.ctl, gridDim.x);  // termination / next iteration
    // write-through of the candidates (host readers: mgfwa_get_candidates)
    // once, after the launch's last generation — no store drain before the
    // cluster barriers of every generation (small_b_body reads none of them)
    if (SM && (gen + 1 == max_gens || *(volatile int*)&v.ctl->active == 0)) {
      copy_words(v.sparks + f * v.lam * v.Dp, w.sparks + f * v.lam * v.Dp, v.lam * v.Dp);
      copy_words(v.spart + f * v.lam * v.nparts * 2, w.spart + f * v.lam * v.nparts * 2, v.lam * v.nparts * 2);
      copy_words(v.guides + f * v.M * v.Dp, w.guides + f * v.M * v.Dp, v.M * v.Dp);
      copy_words(v.gpart + f * v.M * 2, w.gpart + f * v.M * 2, v.M * 2);
      copy_words(v.sfit + f * v.lam, w.sfit + f * v.lam, v.lam);
      copy_words(v.gfit + f * v.M, w.gfit + f * v.M, v.M);
    }
  }
}

static bool small_path_disabled();

bool small_run_ok(const EngineView& v, int nsm) {
  static const bool off = [] {  // MGFWA_SMALL_RUN=0: the graph-replayed kernels instead
    const char* e = getenv("MGFWA_SMALL_RUN");
    return e != nullptr && e[0] == '0';
  }();
  if (off || small_path_disabled()) return false;
  return !v.nn && v.Fl == v.F && v.D <= (uint64_t)kChunk && v.lam <= 2048 && v.top <= 1024 &&
         v.M <= 16 && v.F <= (uint64_t)nsm;
}

static size_t small_run_smem(const EngineView& v, bool sm) {
  return sizeof(ExplodeChunk) + kSmallRunWarps * sizeof(ExplodeWarp) + ((v.lam + 1) & ~1ull) * sizeof(uint64_t) +
         (sm ? small_smem_layout(v).total : 0);
}
#ifndef SMALL_SMEM
#define SMALL_SMEM 1  // cluster form: candidates resident in shared memory when they fit
#endif
constexpr size_t kSmallSmemMax = 200 * 1024;

#ifndef SMALL_CLUSTER
#define SMALL_CLUSTER 1  // F <= 8: one thread-block cluster with the hardware cluster barrier
#endif
cudaError_t launch_small_run(const EngineView& v, uint64_t max_gens, cudaStream_t s) {
  const bool cl = SMALL_CLUSTER && v.F <= 8;
  const bool sm = cl && SMALL_SMEM && small_run_smem(v, true) <= kSmallSmemMax;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)v.F);
  cfg.blockDim = dim3(kSmallRunThreads);
  cfg.dynamicSmemBytes = small_run_smem(v, sm);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (cl) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)v.F;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
  } else {
    attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the grid barrier
    attr[0].val.cooperative = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kern) -> cudaError_t {
    // (the default dynamic limit is 48 KB minus the kernel's static shared memory)
    const cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
    if (e != cudaSuccess) return e;
    return cudaLaunchKernelEx(&cfg, kern, v, max_gens);
  };
  cudaError_t e;
  switch (v.obj_kind) {
    case OBJ_SPHERE:
      e = sm ? go(k_small_run<OBJ_SPHERE, true, true>)
             : cl ? go(k_small_run<OBJ_SPHERE, true, false>) : go(k_small_run<OBJ_SPHERE, false, false>);
      break;
    case OBJ_RASTRIGIN:
      e = sm ? go(k_small_run<OBJ_RASTRIGIN, true, true>)
             : cl ? go(k_small_run<OBJ_RASTRIGIN, true, false>) : go(k_small_run<OBJ_RASTRIGIN, false, false>);
      break;
    default:
      e = sm ? go(k_small_run<OBJ_ACKLEY, true, true>)
             : cl ? go(k_small_run<OBJ_ACKLEY, true, false>) : go(k_small_run<OBJ_ACKLEY, false, false>);
      break;
  }
  if (e != cudaSuccess && cl) {
    // a cluster this size cannot be scheduled here: the cooperative grid form
    (void)cudaGetLastError();
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.dynamicSmemBytes = small_run_smem(v, false);
    switch (v.obj_kind) {
      case OBJ_SPHERE: e = go(k_small_run<OBJ_SPHERE, false, false>); break;
      case OBJ_RASTRIGIN: e = go(k_small_run<OBJ_RASTRIGIN, false, false>); break;
      default: e = go(k_small_run<OBJ_ACKLEY, false, false>); break;
    }
  }
  return e;
}

static bool small_path_disabled() {  // MGFWA_SMALL_PATH=0: always the general kernels
  static const bool off = [] {
    const char* e = getenv("MGFWA_SMALL_PATH");
    return e != nullptr && e[0] == '0';
  }();
  return off;
}

bool small_path(const EngineView& v) {
  return !v.nn && v.Fl == v.F && v.D <= (uint64_t)kChunk && v.lam <= 2048 && v.top <= 1024 &&
         v.M <= 16 && v.mu <= 1024;
}

// ------------------------------------------------------- operator seams
// Analytic partial sums of arbitrary fp32 rows (batched_apply seam).
__global__ void __launch_bounds__(256) k_analytic_partials(const float* rows,
                                                          uint64_t nrows,
                                                          uint64_t D,
                                                          uint64_t Dp,
                                                          uint32_t nch,
                                                          int kind,
                                                          float* part) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const uint64_t items = nrows * nch;
  for (uint64_t item = blockIdx.x * (uint64_t)kWarps + (threadIdx.x >> 5);
       item < items; item += (uint64_t)gridDim.x * kWarps) {
    const uint64_t r = item / nch, c = item % nch;
    float s0 = 0.0f, s1 = 0.0f;
    for (int q = 0; q < 4; ++q) {
      const uint64_t d0 = c * kChunk + q * 128 + lane * 4;
      if (d0 >= D) break;
      const float4 x4 = *reinterpret_cast<const float4*>(rows + r * Dp + d0);
      const float xs[4] = {x4.x, x4.y, x4.z, x4.w};
      // same grouping as the generating kernels: per-4 group, then chunk
      float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (d0 + e < D) analytic_terms(kind, xs[e], a0, a1);
      s0 += a0;
      s1 += a1;
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if (lane == 0) {
      part[(r * nch + c) * 2] = s0;
      part[(r * nch + c) * 2 + 1] = s1;
    }
  }
}

// fitness[r] = finalize(part[r]) with NaN -> +inf; *nan += #NaN.
__global__ void k_finalize_rows(EngineView v, const float* part, uint64_t nrows,
                                float* fitness, unsigned long long* nan) {
  pdl_enter();
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < nrows;
       r += warps) {  // one warp per row
    bool isnan_;
    const float x = finalize_row(v, part, r, &isnan_);
    if ((threadIdx.x & 31) == 0) {
      fitness[r] = x;
      if (isnan_) atomicAdd(nan, 1ull);
    }
  }
}

// fp32 rows -> bf16 rows (tensor-core operand), padding untouched.
__global__ void k_to_bf16(const float* src, __nv_bfloat16* dst, uint64_t n) {
  pdl_enter();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

// Standalone random_mapping over given rows (engine.cpp:103-131); shares
// map_coord with the fused kernels.  cand/out [B][rows][Dp], pop from v.pos.
__global__ void k_map_rows(EngineView v, const float* cand, float* out,
                           uint64_t rows, uint64_t per, uint64_t stream,
                           uint64_t it) {
  pdl_enter();
  const uint64_t total = v.B * rows * v.D;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = i % v.D, r = (i / v.D) % rows, b = i / (v.D * rows);
    const uint64_t n = r / per, k = r % per;
    const uint64_t pm = key_prefix(v.seed, stream, it, b, n, k);
    const float x = cand[(b * rows + r) * v.Dp + d];
    out[(b * rows + r) * v.Dp + d] =
        map_coord(v, (double)x, d, pm, v.pop_lo + b * v.Dp, v.pop_hi + b * v.Dp);
  }
}

// argmin_per_population (backend.cpp:69-83): strict <, lowest index wins.
__global__ void k_argmin_rows(const double* fit, uint64_t rows, uint64_t cols,
                              uint64_t* idx, double* val) {
  pdl_enter();
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < rows;
       b += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t bi = 0;
    double bv = fit[b * cols];
    for (uint64_t n = 1; n < cols; ++n)
      if (fit[b * cols + n] < bv) bv = fit[b * cols + n], bi = n;
    idx[b] = bi;
    val[b] = bv;
  }
}

// key_hash (rng.hpp:43-52) for n keys [n][7].
__global__ void k_key_hash(const uint64_t* keys, uint64_t n, uint64_t* out) {
  pdl_enter();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t* k = keys + 7 * i;
    out[i] = splitmix64(key_prefix(k[0], k[1], k[2], k[3], k[4], k[5]) ^ k[6]);
  }
}

void launch_map_rows(const EngineView& v, const float* cand, float* out,
                     uint64_t rows, uint64_t per, uint64_t stream, uint64_t it,
                     cudaStream_t s) {
  const uint64_t total = v.B * rows * v.D;
  const unsigned g = (unsigned)((total + 255) / 256);
  pdl_launch(k_map_rows, g < 4096 ? (g ? g : 1) : 4096, 256, 0, s, v, cand, out, rows, per, stream, it);
}

void launch_argmin_rows(const double* fit, uint64_t rows, uint64_t cols,
                        uint64_t* idx, double* val, cudaStream_t s) {
  pdl_launch(k_argmin_rows, (unsigned)((rows + 127) / 128), 128, 0, s, fit, rows, cols, idx, val);
}

void launch_key_hash(const uint64_t* keys, uint64_t n, uint64_t* out,
                     cudaStream_t s) {
  pdl_launch(k_key_hash, (unsigned)((n + 255) / 256), 256, 0, s, keys, n, out);
}

// ---------------------------------------------------------------- launch

static size_t guides_smem(const EngineView& v) { return v.M * sizeof(uint64_t) + 2 * v.top * sizeof(int); }

static unsigned guide_blocks(const EngineView& v, int nsm);
static void launch_guides_k(const EngineView& v, int nsm, cudaStream_t s) {
  if (v.top <= 64)
    pdl_launch(k_guides<30>, guide_blocks(v, nsm), kGuideWarps * 32, guides_smem(v), s, v);
  else
    pdl_launch(k_guides<16>, guide_blocks(v, nsm), kGuideWarps * 32, guides_smem(v), s, v);
}
static unsigned guide_blocks(const EngineView& v, int nsm) {
  const uint64_t nsl = (v.D + 32 * GUIDES_VEC - 1) / (32 * GUIDES_VEC);
  const uint64_t blocks = v.Fl * ((nsl + kGuideWarps - 1) / kGuideWarps);
#ifndef GUIDES_CAP_MULT
#define GUIDES_CAP_MULT 64  // measured: C5 guides 3.37 -> 3.17 ms vs 8
#endif
  const uint64_t cap = (uint64_t)nsm * GUIDES_CAP_MULT;
  return (unsigned)(blocks < cap ? (blocks ? blocks : 1) : cap);
}

// k_select blocks per firework: enough to spread the winner-row copy over the
// SMs (about 8 KB per block), at most 16.
static unsigned select_parts(const EngineView& v, int nsm) {
  const uint64_t n4 = (v.D + 3) / 4;
  uint64_t p = (n4 + 511) / 512;
  const uint64_t cap = ((uint64_t)nsm * 4 + v.Fl - 1) / v.Fl;
  p = p < cap ? p : cap;
  p = p < 16 ? p : 16;
  return (unsigned)(p ? p : 1);
}

static unsigned capped(uint64_t g, int nsm) {
  const uint64_t c = (uint64_t)nsm * 16;
  return (unsigned)(g == 0 ? 1 : (g < c ? g : c));
}

// phase kGenAll: the whole loop body; kGenA: pop range .. selection (owned
// fireworks); kGenB: loser-out .. record_wave (all fireworks, after the
// per-generation all-gather of the selected fireworks).
void launch_generation_kernels(const EngineView& v, int nsm, cudaStream_t s,
                               GenerationHooks* hooks, int phase) {
  if (phase == kGenAll && small_path(v) && !small_path_disabled()) {
    launch_explode_map_impl(v, nsm, s);
    pdl_launch(k_small_a, (unsigned)v.Fl, kSmallThreads, v.lam * sizeof(uint64_t), s, v);
    pdl_launch(k_small_b, (unsigned)v.B, kSmallThreads, 0, s, v);
    return;
  }
  if (phase != kGenB) {
    // population_range of this generation was computed by the previous
    // generation's (or initialize's) tail kernel, k_record_copy.
    if (v.nn && hooks->explode_eval) {
      hooks->explode_eval(hooks->ctx, s);  // pipelined: explode chunk c+1 beside fitness chunk c
    } else {
      launch_explode_map_impl(v, nsm, s);
      if (v.nn) hooks->eval_sparks(hooks->ctx, s);
    }
    pdl_launch(k_rank, (unsigned)v.Fl, rank_threads(v), rank_smem(v), s, v);
    if (v.M > 0) {
      launch_guides_k(v, nsm, s);
      if (v.nn)
        hooks->eval_guides(hooks->ctx, s);
      else
        launch_analytic_partials(v.guides, v.Fl * v.M, v.D, v.Dp, v.nch, v.obj_kind, v.gpart, nsm, s);
    }
    pdl_launch(k_select, dim3((unsigned)v.Fl, select_parts(v, nsm)), kSelectThreads, 0, s, v);
  }
  // replica sharding: loser-out (own batches) closes phase A, the loser
  // counts are exchanged, phase B starts at the reinit
  if (v.replica ? phase != kGenB : phase != kGenA) pdl_launch(k_loser, 1, 128, 0, s, v);
  if (phase != kGenA) {
    pdl_launch(k_fresh_rows, capped((v.F * v.nch + kWarps - 1) / kWarps, nsm), 256, 0, s, v, 1);
    if (v.nn) hooks->eval_fresh(hooks->ctx, s);
    pdl_launch(k_finalize_record, 1, 256, 0, s, v, 1);
    pdl_launch(k_record_copy, tail_blocks(v, nsm), 256, 0, s, v);
  }
}

void launch_initialize_kernels(const EngineView& v, int nsm, cudaStream_t s,
                               GenerationHooks* hooks) {
  const unsigned items_f = (unsigned)((v.F * v.nch + kWarps - 1) / kWarps);
  auto cap = [&](unsigned g) { return g < (unsigned)nsm * 16 ? (g ? g : 1) : (unsigned)nsm * 16; };
  pdl_launch(k_fresh_rows, cap(items_f), 256, 0, s, v, 0);
  if (v.nn) hooks->eval_fresh_all(hooks->ctx, s);
  pdl_launch(k_finalize_record, 1, 256, 0, s, v, 0);
  pdl_launch(k_record_copy, tail_blocks(v, nsm), 256, 0, s, v);
}

void launch_analytic_partials(const float* rows, uint64_t nrows, uint64_t D,
                              uint64_t Dp, uint32_t nch, int kind, float* part,
                              int nsm, cudaStream_t s) {
  const unsigned g = (unsigned)((nrows * nch + kWarps - 1) / kWarps);
  pdl_launch(k_analytic_partials, g < (unsigned)nsm * 16 ? (g ? g : 1) : nsm * 16, 256, 0, s, 
      rows, nrows, D, Dp, nch, kind, part);
}

void launch_finalize_rows(const EngineView& v, const float* part, uint64_t nrows,
                          float* fitness, unsigned long long* nan, cudaStream_t s) {
  pdl_launch(k_finalize_rows, (unsigned)((nrows + 7) / 8), 256, 0, s, v, part, nrows, fitness, nan);
}

void launch_add_losers(Ctl* dst, const Ctl* src, int losers, cudaStream_t s) {
  k_add_losers<<<1, 1, 0, s>>>(dst, src, losers);
}

void launch_to_bf16(const float* src, __nv_bfloat16* dst, uint64_t n, cudaStream_t s) {
  pdl_launch(k_to_bf16, (unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, s, src, dst, n);
}

// Individual kernels for the operator seams (tests).
void launch_pop_range(const EngineView& v, int nsm, cudaStream_t s) {
  const unsigned g = (unsigned)((v.B * v.D + 255) / 256);
  pdl_launch(k_pop_range, g < (unsigned)nsm * 16 ? g : nsm * 16, 256, 0, s, v);
}
void launch_explode_map(const EngineView& v, int nsm, cudaStream_t s) {
  const unsigned g = (unsigned)((v.F * ((v.lam + kSparkGroup - 1) / kSparkGroup) * v.nch + kWarps - 1) / kWarps);
  (void)g;
  launch_explode_map_impl(v, nsm, s);
}
void launch_rank(const EngineView& v, cudaStream_t s) {
  pdl_launch(k_rank, (unsigned)v.Fl, rank_threads(v), rank_smem(v), s, v);
}
void launch_guides(const EngineView& v, int nsm, cudaStream_t s) {
  launch_guides_k(v, nsm, s);
  if (!v.nn) launch_analytic_partials(v.guides, v.Fl * v.M, v.D, v.Dp, v.nch, v.obj_kind, v.gpart, nsm, s);
}
void launch_select(const EngineView& v, int nsm, cudaStream_t s) {
  (void)nsm;
  pdl_launch(k_select, (unsigned)v.Fl, kSelectThreads, 0, s, v);
}
// The generation's multi-part k_select (needs k_rank's fit_prev).
void launch_select_gen(const EngineView& v, int nsm, cudaStream_t s) {
  pdl_launch(k_select, dim3((unsigned)v.Fl, select_parts(v, nsm)), kSelectThreads, 0, s, v);
}
void launch_loser(const EngineView& v, int nsm, cudaStream_t s) {
  const unsigned g = (unsigned)((v.F * v.nch + kWarps - 1) / kWarps);
  pdl_launch(k_loser, 1, 128, 0, s, v);
  pdl_launch(k_fresh_rows, g < (unsigned)nsm * 16 ? g : nsm * 16, 256, 0, s, v, 1);
}
void launch_loser_commit(const EngineView& v, int nsm, cudaStream_t s) {
  pdl_launch(k_finalize_record, 1, 256, 0, s, v, 1);
  pdl_launch(k_record_copy, tail_blocks(v, nsm), 256, 0, s, v);
}

}  // namespace mgfwa_b200
