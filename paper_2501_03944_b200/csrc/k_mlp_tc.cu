// k_mlp_tc.cu — population-batched MLP-weights fitness entirely on the
// 5th-gen tensor cores (tcgen05.mma kind::f16, bf16 x bf16 -> fp32 in TMEM).
//
// Objective (builder-defined, pattern nets.cpp:138-167): candidate w holds
// W1[H][I], b1[H], W2[O][H], b2[O] (reference Layer order, nets.hpp:60-65);
// f(w) = mean_s CE(softmax(W2 relu(W1 x_s + b1) + b2), y_s) over S samples.
//
// Layer 1 for the whole population is one GEMM:
//   D1[s][(p,h)] = sum_i X[s][i] * W1_p[h][i]
//   M = samples (128-row tiles = TMEM lanes), N = (spark, hidden) (256 =
//   256/H sparks), K = I (784 = 12 x 64 + 16).  Both operands are K-major —
//   exactly the reference weight layout — and are staged by TMA with the
//   128-byte swizzle; W1 is read straight out of the bf16 spark matrix
//   through a 3-D tensor map (i, h, spark): no repacking pass.
// Layer 2 also runs on the tensor cores: the epilogue turns each fp32 D1
//   column block into bf16 ReLU(D1 + b1) and writes it back into the SAME
//   TMEM columns (tcgen05.st), then one tcgen05.mma per spark with the A
//   operand read from TMEM (M = 128 samples, N = 16 >= O outputs, K = H) and
//   W2^T staged in shared memory produces the logits next to it.  The CUDA
//   cores only do +b1/ReLU/pack and the log-softmax CE.
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer (X 128x64 + W1 256x64 per stage, 4 stages)
//   warp 1      MMA issuer (one thread): layer-1 k-steps of tile t, with the
//               layer-2 MMAs of tile t-1 slotted in as soon as its
//               activations are in TMEM (non-blocking barrier probe)
//   warp 2      TMEM allocator (512 columns = 2 tile buffers)
//   warps 4-11  epilogue
// Output: part[p][m_tile][0] = sum of CE over the m-tile's samples (the
// deterministic finalize divides by S).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_glue.cuh"

namespace mgfwa_b200 {

namespace {

constexpr int BM = 128;  // samples per tile (TMEM lanes)
constexpr int BN = 256;  // (spark, hidden) columns per tile (BNT: the kernel's tile width)
constexpr int BN_NARROW = 64;  // narrow tile for few-row launches (guides, losers; H == 32)
constexpr int BK = 64;   // K per pipeline stage (one 128-byte swizzle atom)
#ifndef MLP_STAGES
#define MLP_STAGES 4
#endif
#ifndef MLP_FAST_MATH
#define MLP_FAST_MATH 1  // CE with the MUFU exp2/log2 forms (__expf/__logf)
#endif
#if MLP_FAST_MATH
#define MLP_EXPF __expf
#define MLP_LOGF __logf
#else
#define MLP_EXPF expf
#define MLP_LOGF logf
#endif
#ifndef MLP_L2_WARP
#define MLP_L2_WARP 1  // layer-2 MMAs issued by warp 3 (0: interleaved into the layer-1 k-loop)
#endif
constexpr bool kL2Warp = MLP_L2_WARP != 0;
#ifndef MLP_L2_PREFETCH
#define MLP_L2_PREFETCH 0  // 1: TMA L2 prefetch of the next N tile's W1 (measured slower: C2 fitness 90.3 -> 93.7 us cold)
#endif
#ifndef MLP_CG2_STAGES
#define MLP_CG2_STAGES 6
#endif
#ifndef MLP_PROBE
#define MLP_PROBE 0  // 1: profiling probe, TMA + layer-1 MMA pipeline only (no epilogue math)
#endif
constexpr int kStages = MLP_STAGES;
constexpr int kABytes = BM * BK * 2;  // 16 KB
// CG = CTA group: 1 (one SM per tile, M = 128) or 2 (an SM pair per tile,
// M = 256, cta_group::2: each CTA stages its own 128 A rows and HALF of B,
// which halves the per-SM operand traffic through shared memory and L2).
template <int CG, int BNT = BN>
struct Cfg {
  static constexpr int kBRows = BNT / CG;                // B rows staged per CTA
  static constexpr int kBBytes = kBRows * BK * 2;        // 32 KB | 16 KB (BNT = 256)
  static constexpr int kStageBytes = kABytes + kBBytes;  // 48 KB | 32 KB
  static constexpr int kStages = CG == 2 ? MLP_CG2_STAGES : BNT < BN ? 6 : MLP_STAGES;
  static constexpr int kO2 = 16 / CG;                    // layer-2 B rows (outputs) per CTA
};
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kN2 = 16;  // layer-2 MMA N (outputs padded to 16)
constexpr int kMaxO = 10;

template <int CG, int BNT = BN>
struct SmemLayoutT {
  static constexpr int kStages = Cfg<CG, BNT>::kStages;
  static constexpr int w2 = kStages * Cfg<CG, BNT>::kStageBytes;  // bf16 W2^T, [spark][kO2][H] interleaved
  static constexpr int b1 = w2 + Cfg<CG, BNT>::kO2 * BNT * 2;  // float[BNT]
  static constexpr int b2 = b1 + BNT * 4;                // float[8][kN2]
  static constexpr int red = b2 + 8 * kN2 * 4;           // float[kEpiWarps][8]
  static constexpr int bars = red + kEpiWarps * 8 * 4;   // u64 barriers
  static constexpr int nbars = 2 * kStages + 8;
  static constexpr int tmem_slot = bars + nbars * 8;
  static constexpr int total = tmem_slot + 16;
};
template <int CG, int BNT = BN>
constexpr int smem_bytes() { return SmemLayoutT<CG, BNT>::total; }

struct MlpArgs {
  uint32_t S, I, H, O;
  uint64_t rows, Dp;
  uint32_t m_tiles, n_tiles, k_blocks, spt;  // spt = sparks per N tile
  const __nv_bfloat16* W;
  const int32_t* y;
  float* part;
  const int* gate;
};

using namespace tc;

// ---- CTA-pair (cta_group::2) variants
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on an mbarrier of (possibly) the peer CTA (shared::cluster address)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cbar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cbar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_test_cluster(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// 2-SM TMA: the completion bytes go to the leader CTA's mbarrier (cbar is a
// shared::cluster address, possibly in the peer CTA).
__device__ __forceinline__ void tma_load_2d_cg2(uint32_t dst, const CUtensorMap* map, uint32_t cbar,
                                                int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(cbar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_cg2(uint32_t dst, const CUtensorMap* map, uint32_t cbar,
                                                int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(cbar), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void mma_ss2(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_ts2(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}
// commit to the same barrier offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit2(uint32_t bar) {
  const uint16_t mask = 3;
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}

__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
}

// ----------------------------------------------------- TMEM column plan
// Tile buffer (256 columns).  Spark j of the tile owns D1 columns
// [j*H, (j+1)*H).  After the epilogue has read them, its bf16 activations
// (H values = H/2 columns) and its 16 logit columns are placed inside that
// same range, so no column is written before its owner warp has read it:
//   H <= 128: A2 at [jH, jH + H/2), D2 at [jH + H/2, jH + H/2 + 16)
//   H == 256: A2 halves at [0, 64) and [128, 192) (one per column half),
//             D2 at [64, 80)
template <int H>
__device__ __forceinline__ uint32_t a2_col(int n0) {  // packed column of D1 column n0
  if (H <= 128) return (uint32_t)((n0 / H) * H + (n0 % H) / 2);
  return (uint32_t)((n0 / 128) * 128 + (n0 % 128) / 2);
}
template <int H>
__device__ __forceinline__ uint32_t a2_kcol(int j, int kk) {  // A column of K16 step kk
  if (H <= 128) return (uint32_t)(j * H + kk * 8);
  return (uint32_t)((kk < 8 ? 0 : 128) + (kk & 7) * 8);
}
template <int H>
__device__ __forceinline__ uint32_t d2_col(int j) {
  if (H <= 128) return (uint32_t)(j * H + H / 2);
  return 64u;
}

// ------------------------------------------------------------------ kernel
template <int H, int CG, int BNT = BN>
__global__ void __launch_bounds__(kThreads, 1)
    k_mlp_fitness(const __grid_constant__ CUtensorMap tmap_x,
                  const __grid_constant__ CUtensorMap tmap_w, MlpArgs args) {
  pdl_enter();
  if (args.gate != nullptr && *args.gate == 0) return;
  constexpr int SPT = BNT / H;  // sparks per N tile (1 when H == BNT)
  static_assert(BNT % H == 0 && H % 32 == 0, "H must divide the tile width and be a multiple of 32");
  static_assert(BNT == BN || (CG == 1 && SPT == 2), "narrow tiles: one spark per column half");
  constexpr int kHalf = BNT / 2;        // epilogue column half
  constexpr int kTmemCols = 2 * BNT;    // two tile buffers
  using SmemLayout = SmemLayoutT<CG, BNT>;
  constexpr int kStages = Cfg<CG, BNT>::kStages;
  constexpr int kStageBytes = Cfg<CG, BNT>::kStageBytes;
  constexpr int kO2 = Cfg<CG, BNT>::kO2;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0u;  // CTA rank in the pair
  const bool leader = rank == 0;

  // 1024-byte aligned (SWIZZLE_128B atoms); no static shared memory is used,
  // so the dynamic window starts at the aligned base.
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* s_w2 = smem + SmemLayout::w2;
  float* s_b1 = reinterpret_cast<float*>(smem + SmemLayout::b1);
  float* s_b2 = reinterpret_cast<float*>(smem + SmemLayout::b2);
  float* s_red = reinterpret_cast<float*>(smem + SmemLayout::red);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SmemLayout::bars);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SmemLayout::tmem_slot);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t bar_full = smem_u32(bars);
  const uint32_t bar_empty = smem_u32(bars + kStages);
  const uint32_t bar_tfull = smem_u32(bars + 2 * kStages);       // D1 ready
  const uint32_t bar_tempty = smem_u32(bars + 2 * kStages + 2);  // buffer free
  const uint32_t bar_a2full = smem_u32(bars + 2 * kStages + 4);  // activations in TMEM
  const uint32_t bar_d2full = smem_u32(bars + 2 * kStages + 6);  // logits ready

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(bar_full + 8 * i, 1);
      mbar_init(bar_empty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_tfull + 8 * i, 1);
      mbar_init(bar_tempty + 8 * i, kEpiWarps * CG);  // CG == 2: both CTAs' epilogues (leader's)
      mbar_init(bar_a2full + 8 * i, kEpiWarps * CG);
      mbar_init(bar_d2full + 8 * i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_w)));
  }
  if (warp == 2) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
          smem_u32(tmem_slot)), "n"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
          smem_u32(tmem_slot)), "n"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync_all();  // peer barriers initialised, TMEM allocated on both SMs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the leader's copies of the pipeline barriers (TMA completion, epilogue arrivals)
  const uint32_t c_full = CG == 2 ? mapa_rank(bar_full, 0) : bar_full;
  const uint32_t c_tempty = CG == 2 ? mapa_rank(bar_tempty, 0) : bar_tempty;
  const uint32_t c_a2full = CG == 2 ? mapa_rank(bar_a2full, 0) : bar_a2full;

  // Static contiguous tile range per CTA: tile t -> (n_tile = t / m_tiles,
  // m_tile = t % m_tiles), so one CTA walks all m-tiles of an N tile in turn
  // (its W1 tile stays hot in L2; X is L2-resident for everyone).
  // CG == 2: a unit is (n-tile, m-tile pair); CTA `rank` takes m-tile 2 mp + rank.
  const uint32_t m_units = CG == 2 ? (args.m_tiles + 1) / 2 : args.m_tiles;
  const uint32_t total = m_units * args.n_tiles;
  const uint32_t groups = gridDim.x / CG, group = blockIdx.x / CG;
  const uint32_t t_begin = (uint32_t)(((uint64_t)total * group) / groups);
  const uint32_t t_end = (uint32_t)(((uint64_t)total * (group + 1)) / groups);

  constexpr uint32_t idesc2_l2 = idesc_bf16(BM * CG, kN2);
  const uint32_t w2_base = smem_u32(s_w2);
  // layer-2 MMAs of the tile whose activations sit in buffer `b`
  auto issue_layer2_t = [&](uint32_t b) {
    tc_fence_after();
    const uint32_t cb = tmem_base + b * BNT;
#pragma unroll
    for (int j = 0; j < (MLP_PROBE == 3 ? 0 : SPT); ++j) {
      const uint32_t bj = w2_base + (uint32_t)(j * kO2 * H * 2);
#pragma unroll
      for (int kk = 0; kk < H / 16; ++kk) {
        // B: kO2 output rows x 16 K per step; core matrices 8 rows x 16 B,
        // K-adjacent ones (kO2/8)*128 B apart, N-adjacent 128 B apart
        const uint64_t bd = interleaved_desc(bj + kk * (kO2 / 8) * 256, (kO2 / 8) * 128, 128);
        if (CG == 2)
          mma_ts2(cb + d2_col<H>(j), cb + a2_kcol<H>(j, kk), bd, idesc2_l2, kk != 0);
        else
          mma_ts(cb + d2_col<H>(j), cb + a2_kcol<H>(j, kk), bd, idesc2_l2, kk != 0);
      }
    }
    if (CG == 2) mma_commit2(bar_d2full + 8 * b); else mma_commit(bar_d2full + 8 * b);
  };
  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = t_begin; t < t_end; ++t) {
        const int m_tile = (int)((t % m_units) * CG + rank), n_tile = (int)(t / m_units);
        // Entering an N tile: pull this CTA's next N tile of W1 into L2 (its
        // first m-tile would otherwise stream it from HBM at TMA latency).
        if (MLP_L2_PREFETCH && (t == t_begin || t % m_units == 0) && (uint32_t)(n_tile + 1) * m_units < t_end) {
          for (uint32_t kb = 0; kb < args.k_blocks; ++kb) {
            if (SPT >= 2)
              tma_prefetch_3d(&tmap_w, (int)(kb * BK), 0, (n_tile + 1) * SPT + (CG == 2 ? (int)rank * (SPT / 2) : 0));
            else
              tma_prefetch_3d(&tmap_w, (int)(kb * BK), CG == 2 ? (int)rank * (H / 2) : 0, n_tile + 1);
          }
        }
        for (uint32_t kb = 0; kb < args.k_blocks; ++kb) {
          mbar_wait(bar_empty + 8 * stage, phase ^ 1);
          const uint32_t sa = smem_u32(smem + stage * kStageBytes);
#if MLP_PROBE == 2  // profiling probe: no operand traffic after the first round of stages
          if (t != t_begin || kb >= (uint32_t)kStages) {
            mbar_arrive(bar_full + 8 * stage);
            if (++stage == kStages) stage = 0, phase ^= 1;
            continue;
          }
#endif
          if (CG == 2) {
            // both CTAs' halves complete on the leader's barrier
            if (leader) mbar_expect_tx(bar_full + 8 * stage, 2 * kStageBytes);
            const uint32_t cb = c_full + 8 * stage;
            tma_load_2d_cg2(sa, &tmap_x, cb, (int)(kb * BK), m_tile * BM);
            if (SPT >= 2)  // this CTA's half of the sparks of the N tile
              tma_load_3d_cg2(sa + kABytes, &tmap_w, cb, (int)(kb * BK), 0,
                              n_tile * SPT + (int)rank * (SPT / 2));
            else  // H == 256: this CTA's half of the hidden rows
              tma_load_3d_cg2(sa + kABytes, &tmap_w, cb, (int)(kb * BK), (int)rank * (H / 2), n_tile);
          } else {
            mbar_expect_tx(bar_full + 8 * stage, kStageBytes);
            tma_load_2d(sa, &tmap_x, bar_full + 8 * stage, (int)(kb * BK), m_tile * BM);
            tma_load_3d(sa + kABytes, &tmap_w, bar_full + 8 * stage, (int)(kb * BK), 0, n_tile * SPT);
          }
          if (++stage == kStages) stage = 0, phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (the leader CTA of a pair)
      constexpr uint32_t idesc1 = idesc_bf16(BM * CG, BNT);
      constexpr uint32_t idesc2 = idesc_bf16(BM * CG, kN2);
      auto mma1 = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
        if (CG == 2) mma_ss2(d, a, b, idesc1, acc); else mma_ss(d, a, b, idesc1, acc);
      };
      auto commit = [&](uint32_t bar) {
        if (CG == 2) mma_commit2(bar); else mma_commit(bar);
      };
      auto a2ready = [&](uint32_t b, uint32_t u) {
        return CG == 2 ? mbar_test_cluster(bar_a2full + 8 * b, u) : mbar_test(bar_a2full + 8 * b, u);
      };
      auto a2wait = [&](uint32_t b, uint32_t u) {
        if (CG == 2) mbar_wait_cluster(bar_a2full + 8 * b, u); else mbar_wait(bar_a2full + 8 * b, u);
      };
      auto issue_layer2 = [&](uint32_t b) { issue_layer2_t(b); };
      uint32_t stage = 0, phase = 0, i = 0;
      bool pend = false;
      uint32_t pbuf = 0, puse = 0;
      for (uint32_t t = t_begin; t < t_end; ++t, ++i) {
        const uint32_t buf = i & 1, use = (i >> 1) & 1;
        if (CG == 2) mbar_wait_cluster(bar_tempty + 8 * buf, use ^ 1);
        else mbar_wait(bar_tempty + 8 * buf, use ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * BNT;
        for (uint32_t kb = 0; kb < args.k_blocks; ++kb) {
          mbar_wait(bar_full + 8 * stage, phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kStageBytes);
          const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + kABytes);
          const uint32_t rem = args.I - kb * BK;
          const uint32_t nk = rem >= BK ? BK / 16 : (rem + 15) / 16;
          for (uint32_t kk = 0; kk < nk; ++kk) mma1(d_tmem, da + 2 * kk, db + 2 * kk, (kb | kk) != 0);
          commit(bar_empty + 8 * stage);
          if (++stage == kStages) stage = 0, phase ^= 1;
          if (!kL2Warp && pend && a2ready(pbuf, puse)) {
            issue_layer2(pbuf);
            pend = false;
          }
        }
        commit(bar_tfull + 8 * buf);
        if (kL2Warp || MLP_PROBE == 1 || MLP_PROBE == 2) continue;
        if (pend) {
          a2wait(pbuf, puse);
          issue_layer2(pbuf);
        }
        pend = true;
        pbuf = buf;
        puse = use;
      }
      if (!kL2Warp && pend && MLP_PROBE != 1 && MLP_PROBE != 2) {
        a2wait(pbuf, puse);
        issue_layer2(pbuf);
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    if (kL2Warp && lane == 0 && leader && MLP_PROBE != 1 && MLP_PROBE != 2) {
      // ---------------- layer-2 MMA issuer: as soon as tile t's activations
      // are in TMEM (independent of the layer-1 k-loop's TMA waits)
      uint32_t i = 0;
      for (uint32_t t = t_begin; t < t_end; ++t, ++i) {
        const uint32_t buf = i & 1, use = (i >> 1) & 1;
        if (CG == 2) mbar_wait_cluster(bar_a2full + 8 * buf, use); else mbar_wait(bar_a2full + 8 * buf, use);
        issue_layer2_t(buf);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------- epilogue
    const int e = warp - 4;            // 0..7
    const int q = warp & 3;            // TMEM lane quarter (warp % 4)
    const int half = e >> 2;           // D1 column half: [half*kHalf, (half+1)*kHalf)
    const int row = q * 32 + lane;     // accumulator row == sample within tile
    const int et = threadIdx.x - 128;  // 0..255
    const uint32_t O = args.O;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    uint32_t i = 0;
    uint32_t staged_n = 0xFFFFFFFFu;
    for (uint32_t t = t_begin; t < t_end; ++t, ++i) {
      const uint32_t m_tile = (t % m_units) * CG + rank, n_tile = t / m_units;
      const uint32_t buf = i & 1, use = (i >> 1) & 1;
      const uint32_t cb = tmem_base + buf * BNT + lane_off;
      const uint32_t s = m_tile * BM + row;
      const bool valid = s < args.S;
      const int label = valid ? args.y[s] : 0;
      if (MLP_PROBE == 1 || MLP_PROBE == 2) {
        mbar_wait(bar_tfull + 8 * buf, use);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2) mbar_arrive_cluster(c_tempty + 8 * buf); else mbar_arrive(bar_tempty + 8 * buf);
        }
        continue;
      }
      // Stage b1 (fp32), b2 (fp32) and W2^T (bf16, interleaved core-matrix
      // layout: element (o, h) of spark j at j*16*H*2 + ((h/8)*2 + o/8)*128
      // + (o%8)*16 + (h%8)*2) when the N tile changes (every m_tiles tiles).
      // The previous tile's layer-2 MMAs finished before this warp group
      // passed its logits barrier, and the barrier below orders s_red.
      epi_bar();
      if (n_tile != staged_n) {
      staged_n = n_tile;
      for (int idx = et; idx < SPT * H; idx += kEpiThreads) {
        const int j = idx / H, h = idx % H;
        const uint64_t p = (uint64_t)n_tile * SPT + j;
        const bool ok = p < args.rows;
        const __nv_bfloat16* base = args.W + (ok ? p : 0) * args.Dp + (uint64_t)H * args.I;
        s_b1[idx] = ok ? __bfloat162float(base[h]) : 0.0f;
        __nv_bfloat16* w2j = reinterpret_cast<__nv_bfloat16*>(s_w2 + j * kO2 * H * 2);
#pragma unroll
        for (int ol = 0; ol < kO2; ++ol) {  // this CTA's output rows o = rank * kO2 + ol
          const int o = (int)rank * kO2 + ol;
          const __nv_bfloat16 wv =
              (ok && (uint32_t)o < O) ? base[H + o * H + h] : __float2bfloat16_rn(0.0f);
          w2j[(((h >> 3) * (kO2 / 8) + (ol >> 3)) * 128 + (ol & 7) * 16 + (h & 7) * 2) / 2] = wv;
        }
      }
      for (int idx = et; idx < SPT * kN2; idx += kEpiThreads) {
        const int j = idx / kN2, o = idx % kN2;
        const uint64_t p = (uint64_t)n_tile * SPT + j;
        float v = 0.0f;
        if (p < args.rows && (uint32_t)o < O)
          v = __bfloat162float(args.W[p * args.Dp + (uint64_t)H * args.I + H + (uint64_t)O * H + o]);
        s_b2[idx] = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // W2 visible to the MMA
      epi_bar();
      }

      // ---- layer-1 epilogue: bf16(ReLU(D1 + b1)) back into TMEM
      mbar_wait(bar_tfull + 8 * buf, use);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < kHalf / 32; ++c) {
        const int col0 = half * kHalf + c * 32;
        float acc[32];
        tmem_ld32(cb + col0, acc);
        uint32_t pk[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const float h0 = fmaxf(acc[2 * u] + s_b1[col0 + 2 * u], 0.0f);
          const float h1 = fmaxf(acc[2 * u + 1] + s_b1[col0 + 2 * u + 1], 0.0f);
          __nv_bfloat162 v2 = __floats2bfloat162_rn(h0, h1);
          pk[u] = *reinterpret_cast<uint32_t*>(&v2);
        }
        tmem_st16(cb + a2_col<H>(col0), pk);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(c_a2full + 8 * buf); else mbar_arrive(bar_a2full + 8 * buf);
      }

      // ---- logits (layer-2 MMA result) -> log-softmax CE
      mbar_wait(bar_d2full + 8 * buf, use);
      tc_fence_after();
      const int jb = H > 128 ? 0 : half * (SPT / 2);
      const int jn = H > 128 ? (half == 0 ? 1 : 0) : SPT / 2;
      constexpr int JN = H > 128 ? 1 : SPT / 2;  // logit blocks per thread (H > 128: half 0 only)
      // all of the thread's logit blocks in flight at once, one wait
      float z[JN][kN2];
#pragma unroll
      for (int jj = 0; jj < JN; ++jj)
        if (jj < jn) tmem_ld16_nowait(cb + d2_col<H>(jb + jj), z[jj]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      // CE of the thread's JN logit blocks as JN interleaved chains (max, exp
      // sums, log, then the warp butterflies stage by stage), the same
      // operation order per block as one block at a time
      float loss[JN];
#pragma unroll
      for (int jj = 0; jj < JN; ++jj) loss[jj] = 0.0f;
      if (valid && jn > 0) {  // jn: warp-uniform (0 only for the second half when H > 128)
        float mx[JN], se[JN], zl[JN];
#pragma unroll
        for (int jj = 0; jj < JN; ++jj) {
          mx[jj] = -INFINITY;
#pragma unroll
          for (int o = 0; o < kMaxO; ++o) {
            z[jj][o] += s_b2[(jb + jj) * kN2 + o];
            if ((uint32_t)o < O) mx[jj] = fmaxf(mx[jj], z[jj][o]);
          }
        }
#pragma unroll
        for (int jj = 0; jj < JN; ++jj) {
          se[jj] = 0.0f;
          zl[jj] = 0.0f;
#pragma unroll
          for (int o = 0; o < kMaxO; ++o) {
            if ((uint32_t)o < O) se[jj] += MLP_EXPF(z[jj][o] - mx[jj]);
            if (o == label) zl[jj] = z[jj][o];
          }
        }
#pragma unroll
        for (int jj = 0; jj < JN; ++jj) loss[jj] = (mx[jj] + MLP_LOGF(se[jj])) - zl[jj];
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int jj = 0; jj < JN; ++jj) loss[jj] += __shfl_xor_sync(0xffffffffu, loss[jj], off);
      if (lane == 0)
#pragma unroll
        for (int jj = 0; jj < JN; ++jj)
          if (jj < jn) s_red[e * 8 + jj] = loss[jj];
      // tile buffer consumed: hand it back to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(c_tempty + 8 * buf); else mbar_arrive(bar_tempty + 8 * buf);
      }
      epi_bar();
      // deterministic per-(spark, m-tile) partial: the 4 lane quarters in order
      if (et < SPT) {
        const int j = et;
        const int hh = H > 128 ? 0 : (j * H) / kHalf;
        const int jl = H > 128 ? 0 : j - hh * (SPT / 2);
        float sum = 0.0f;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) sum += s_red[(hh * 4 + qq) * 8 + jl];
        const uint64_t p = (uint64_t)n_tile * SPT + j;
        if (p < args.rows && m_tile < args.m_tiles) {
          args.part[(p * args.m_tiles + m_tile) * 2] = sum;
          args.part[(p * args.m_tiles + m_tile) * 2 + 1] = 0.0f;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync_all();  // no MMA of the pair targets this TMEM any more
  if (warp == 2) {
    tc_fence_after();
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols));
  }
}

// -------------------------------------------------------------- host side
template <int H, int CG, int BNT = BN>
cudaError_t prepare_h() {
  return cudaFuncSetAttribute(k_mlp_fitness<H, CG, BNT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              smem_bytes<CG, BNT>());
}

template <int H, int CG, int BNT = BN>
cudaError_t launch_h(const CUtensorMap& tx, const CUtensorMap& tw, int grid, const MlpArgs& a,
                     cudaStream_t s, cudaEvent_t launch_done) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes<CG, BNT>();
  cfg.stream = s;
  cudaLaunchAttribute attr[3];
  int n = 0;
  if (launch_done) {
    attr[n].id = cudaLaunchAttributeLaunchCompletionEvent;
    attr[n].val.launchCompletionEvent.event = launch_done;
    attr[n].val.launchCompletionEvent.flags = 0;
    ++n;
  }
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (CG == 2) {  // the SM pair of a tile is a 2-CTA cluster
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = 2;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, k_mlp_fitness<H, CG, BNT>, tx, tw, a);
}

// CTA group of a plan (MGFWA_MLP_CG=1|2 overrides).  Default: the SM pair
// (cta_group::2, M = 256: each CTA stages its own X rows and HALF of the W1
// tile, a third less operand traffic through L2 per MMA) for H >= 128, where
// the kernel is bound by L2 -> shared-memory operand delivery (C5, H = 256:
// 26.7 -> 24.8 ms per generation); one SM per tile for narrower hidden
// layers, where the pair's cross-CTA epilogue handshakes cost more than the
// traffic saves (C2, H = 32: 90.1 vs 103.7 us).
int mlp_cg(uint32_t H) {
  static const int forced = [] {
    const char* e = getenv("MGFWA_MLP_CG");
    if (e && e[0] == '1') return 1;
    if (e && e[0] == '2') return 2;
    return 0;
  }();
  if (forced) return forced;
  return H >= 128 ? 2 : 1;
}

}  // namespace

struct MlpPlan {
  CUtensorMap tmap_x;
  CUtensorMap tmap_w;
  MlpArgs args;
  int grid;
  int H;
  int cg;
  int bnt;  // N tile width: BN, or BN_NARROW for few-row launches
};

uint32_t mlp_num_parts(uint32_t S) { return (S + BM - 1) / BM; }

MlpPlan* mlp_plan_create(const __nv_bfloat16* X, const int32_t* y, uint32_t S, uint32_t I,
                         uint32_t H, uint32_t O, const __nv_bfloat16* W, uint64_t rows,
                         uint64_t Dp, int nsm, char* err, size_t errlen) {
  auto fail = [&](const char* m) -> MlpPlan* {
    if (err && errlen) snprintf(err, errlen, "%s", m);
    return nullptr;
  };
  if (H != 32 && H != 64 && H != 128 && H != 256)
    return fail("MLP fitness: hidden width must be 32, 64, 128 or 256");
  if (O < 2 || O > (uint32_t)kMaxO) return fail("MLP fitness: out_dim must be in [2, 10]");
  if (I % 16 != 0 || I < 16) return fail("MLP fitness: in_dim must be a multiple of 16");
  if ((Dp * 2) % 16 != 0) return fail("MLP fitness: row stride must be 16-byte aligned");
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail("MLP fitness: cuTensorMapEncodeTiled unavailable");
  MlpPlan* p = new MlpPlan();
  memset(p, 0, sizeof(*p));
  {
    cuuint64_t dims[2] = {I, S};
    cuuint64_t strides[1] = {(cuuint64_t)I * 2};
    cuuint32_t box[2] = {BK, BM};
    cuuint32_t es[2] = {1, 1};
    if (enc(&p->tmap_x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(X), dims,
            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      delete p;
      return fail("MLP fitness: X tensor map encode failed");
    }
  }
  const int cg = mlp_cg(H);
  // Few rows (the guides, the loser re-evaluations): narrow 64-column tiles
  // (2 sparks of H = 32) so the launch spreads over more SMs — C2 guides:
  // 15 rows = 16 tiles of 256 columns -> 64 tiles of 64.  MGFWA_MLP_NARROW=0
  // keeps 256-column tiles.
  const uint32_t m_tiles = mlp_num_parts(S);
  const char* nenv = getenv("MGFWA_MLP_NARROW");
  const bool narrow = H == 32 && cg == 1 && !(nenv && nenv[0] == '0') &&
                      2ull * m_tiles * ((rows + BN / H - 1) / (BN / H)) <= (uint64_t)nsm;
  const int bnt = narrow ? BN_NARROW : BN;
  const uint32_t spt = (uint32_t)bnt / H;
  {
    cuuint64_t dims[3] = {I, H, rows};
    cuuint64_t strides[2] = {(cuuint64_t)I * 2, (cuuint64_t)Dp * 2};
    // CG == 2: each CTA stages half of the N tile (half the sparks, or half
    // the hidden rows of the one spark when H == 256)
    cuuint32_t box[3] = {BK, cg == 2 && spt == 1 ? H / 2 : H, cg == 2 && spt >= 2 ? spt / 2 : spt};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&p->tmap_w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<__nv_bfloat16*>(W), dims,
            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      delete p;
      return fail("MLP fitness: W tensor map encode failed");
    }
  }
  p->H = (int)H;
  p->bnt = bnt;
  p->args.S = S;
  p->args.I = I;
  p->args.H = H;
  p->args.O = O;
  p->args.rows = rows;
  p->args.Dp = Dp;
  p->args.m_tiles = mlp_num_parts(S);
  p->args.n_tiles = (uint32_t)((rows + spt - 1) / spt);
  p->args.k_blocks = (I + BK - 1) / BK;
  p->args.spt = spt;
  p->args.W = W;
  p->args.y = y;
  p->cg = cg;
  if (cg == 2) {
    const uint32_t units = ((p->args.m_tiles + 1) / 2) * p->args.n_tiles;
    const uint32_t pairs = (uint32_t)nsm / 2;
    p->grid = 2 * (int)(units < pairs ? units : pairs);
  } else {
    const uint32_t tiles = p->args.m_tiles * p->args.n_tiles;
    p->grid = (int)(tiles < (uint32_t)nsm ? tiles : (uint32_t)nsm);
  }
  const cudaError_t e =
      narrow ? prepare_h<32, 1, BN_NARROW>() :
      cg == 2 ? (H == 32 ? prepare_h<32, 2>() : H == 64 ? prepare_h<64, 2>()
                 : H == 128 ? prepare_h<128, 2>() : prepare_h<256, 2>())
              : (H == 32 ? prepare_h<32, 1>() : H == 64 ? prepare_h<64, 1>()
                 : H == 128 ? prepare_h<128, 1>() : prepare_h<256, 1>());
  if (e != cudaSuccess) {
    delete p;
    return fail(cudaGetErrorString(e));
  }
  return p;
}

void mlp_plan_destroy(MlpPlan* p) { delete p; }

cudaError_t mlp_fitness_launch(const MlpPlan* p, float* part, const int* gate, cudaStream_t s,
                               cudaEvent_t launch_done) {
  MlpArgs a = p->args;
  a.part = part;
  a.gate = gate;
  if (p->bnt == BN_NARROW) return launch_h<32, 1, BN_NARROW>(p->tmap_x, p->tmap_w, p->grid, a, s, launch_done);
  if (p->cg == 2) {
    switch (p->H) {
      case 32: return launch_h<32, 2>(p->tmap_x, p->tmap_w, p->grid, a, s, launch_done);
      case 64: return launch_h<64, 2>(p->tmap_x, p->tmap_w, p->grid, a, s, launch_done);
      case 128: return launch_h<128, 2>(p->tmap_x, p->tmap_w, p->grid, a, s, launch_done);
      case 256: return launch_h<256, 2>(p->tmap_x, p->tmap_w, p->grid, a, s, launch_done);
    }
  }
  switch (p->H) {
    case 32: return launch_h<32, 1>(p->tmap_x, p->tmap_w, p->grid, a, s, launch_done);
    case 64: return launch_h<64, 1>(p->tmap_x, p->tmap_w, p->grid, a, s, launch_done);
    case 128: return launch_h<128, 1>(p->tmap_x, p->tmap_w, p->grid, a, s, launch_done);
    case 256: return launch_h<256, 1>(p->tmap_x, p->tmap_w, p->grid, a, s, launch_done);
  }
  return cudaErrorInvalidValue;
}

}  // namespace mgfwa_b200
