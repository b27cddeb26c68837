// k_mlp_tc.cu — population-batched MLP-weights fitness on the 5th-gen
// tensor cores (tcgen05.mma kind::f16, bf16 x bf16 -> fp32 in TMEM, operands
// staged by TMA with the 128-byte swizzle).
//
// Objective (builder-defined, pattern nets.cpp:138-167): candidate w holds
// W1[H][I], b1[H], W2[O][H], b2[O] (reference Layer order, nets.hpp:60-65);
// f(w) = mean_s CE(softmax(W2 relu(W1 x_s + b1) + b2), y_s) over S samples.
//
// GEMM view of layer 1 for the whole population:
//   D[s][(p,h)] = sum_i X[s][i] * W1_p[h][i]
//   M = samples (tile 128 = TMEM lanes), N = (spark, hidden) (tile 256 =
//   256/H sparks), K = I (784 = 12 x 64 + 16).  Both operands are K-major,
//   which is exactly the reference weight layout (weights[out x in]).
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer (X tile 128x64 + W tile 256x64 per stage, 4 stages)
//   warp 1      MMA issuer (one thread; 4 x tcgen05.mma 128x256x16 per stage)
//   warp 2      TMEM allocator (512 columns = 2 accumulator buffers)
//   warps 4-11  epilogue: tcgen05.ld -> +b1, ReLU -> layer 2 (CUDA cores) ->
//               log-softmax CE -> per-(spark, m-tile) partial loss.
// Double-buffered TMEM lets the epilogue of tile t overlap the MMAs of t+1.
// Output: part[p][m_tile][0] = sum of CE over the m-tile's samples (the
// deterministic finalize divides by S).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include "common.cuh"
#include "kernels.h"

namespace mgfwa_b200 {

namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int kStages = 4;
constexpr int kABytes = BM * BK * 2;  // 16 KB
constexpr int kBBytes = BN * BK * 2;  // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kOPad = 12;  // logits padded to 3 x float4
constexpr int kMaxO = 12;

struct SmemLayout {
  static constexpr int stages = 0;
  static constexpr int b1 = kStages * kStageBytes;           // float[BN]
  static constexpr int w2t = b1 + BN * 4;                    // float[BN][kOPad]
  static constexpr int b2 = w2t + BN * kOPad * 4;            // float[8][kOPad]
  static constexpr int zsh = b2 + 8 * kOPad * 4;             // float[BM][kOPad] (H > 128)
  static constexpr int red = zsh + BM * kOPad * 4;           // float[kEpiWarps][8]
  static constexpr int bars = red + kEpiWarps * 8 * 4;       // u64 barriers
  static constexpr int nbars = 2 * kStages + 4;
  static constexpr int tmem_slot = bars + nbars * 8;
  static constexpr int total = tmem_slot + 16;
};
constexpr int kSmemBytes = SmemLayout::total + 1024;  // + alignment slack

struct MlpArgs {
  uint32_t S, I, H, O;
  uint64_t rows, Dp;
  uint32_t m_tiles, n_tiles, k_blocks, spt;  // spt = sparks per N tile
  const __nv_bfloat16* W;
  const int32_t* y;
  float* part;
  const int* gate;
};

// ---------------------------------------------------------------- PTX glue
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// K-major operand, 128-byte swizzle: rows of 128 B, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;            // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024u >> 4) << 32;  // SBO
  d |= (uint64_t)1u << 46;            // descriptor version (tcgen05)
  d |= (uint64_t)2u << 61;            // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: D=f32, A=B=bf16, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&r)[32]) {
  uint32_t* u = reinterpret_cast<uint32_t*>(r);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
        "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
        "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]),
        "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]),
        "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ------------------------------------------------------------------ kernel
template <int H>
__global__ void __launch_bounds__(kThreads, 1)
    k_mlp_fitness(const __grid_constant__ CUtensorMap tmap_x,
                  const __grid_constant__ CUtensorMap tmap_w, MlpArgs args) {
  if (args.gate != nullptr && *args.gate == 0) return;
  constexpr int SPT = BN / H;  // sparks per N tile (1 when H == 256)
  constexpr bool kSplitSpark = H > 128;
  static_assert(BN % H == 0 && H % 32 == 0, "H must divide 256 and be a multiple of 32");

  // 1024-byte aligned (SWIZZLE_128B atoms); no static shared memory is used,
  // so the dynamic window starts at the aligned base.  Deriving every
  // pointer from this array keeps the accesses in the shared state space
  // (LDS/STS, not generic LD/ST).
  extern __shared__ __align__(1024) uint8_t smem[];
  float* s_b1 = reinterpret_cast<float*>(smem + SmemLayout::b1);
  float* s_w2t = reinterpret_cast<float*>(smem + SmemLayout::w2t);
  float* s_b2 = reinterpret_cast<float*>(smem + SmemLayout::b2);
  float* s_z = reinterpret_cast<float*>(smem + SmemLayout::zsh);
  float* s_red = reinterpret_cast<float*>(smem + SmemLayout::red);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SmemLayout::bars);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SmemLayout::tmem_slot);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t bar_full = smem_u32(bars);
  const uint32_t bar_empty = smem_u32(bars + kStages);
  const uint32_t bar_tfull = smem_u32(bars + 2 * kStages);
  const uint32_t bar_tempty = smem_u32(bars + 2 * kStages + 2);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(bar_full + 8 * i, 1);
      mbar_init(bar_empty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_tfull + 8 * i, 1);
      mbar_init(bar_tempty + 8 * i, kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_x)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_w)));
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // static contiguous tile range per CTA: tile t -> (n_tile = t / m_tiles,
  // m_tile = t % m_tiles), so one CTA walks all m-tiles of an N tile in turn
  // (its W tile stays hot in L2; X is L2-resident for everyone).
  const uint32_t total = args.m_tiles * args.n_tiles;
  const uint32_t t_begin = (uint32_t)(((uint64_t)total * blockIdx.x) / gridDim.x);
  const uint32_t t_end = (uint32_t)(((uint64_t)total * (blockIdx.x + 1)) / gridDim.x);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = t_begin; t < t_end; ++t) {
        const int m_tile = (int)(t % args.m_tiles), n_tile = (int)(t / args.m_tiles);
        for (uint32_t kb = 0; kb < args.k_blocks; ++kb) {
          mbar_wait(bar_empty + 8 * stage, phase ^ 1);
          const uint32_t sa = smem_u32(smem + stage * kStageBytes);
          const uint32_t sb = sa + kABytes;
          mbar_expect_tx(bar_full + 8 * stage, kStageBytes);
          tma_load_2d(sa, &tmap_x, bar_full + 8 * stage, (int)(kb * BK), m_tile * BM);
          tma_load_3d(sb, &tmap_w, bar_full + 8 * stage, (int)(kb * BK), 0, n_tile * SPT);
          if (++stage == kStages) stage = 0, phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16(BM, BN);
      uint32_t stage = 0, phase = 0;
      uint32_t i = 0;
      for (uint32_t t = t_begin; t < t_end; ++t, ++i) {
        const uint32_t buf = i & 1, use = (i >> 1) & 1;
        mbar_wait(bar_tempty + 8 * buf, use ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        for (uint32_t kb = 0; kb < args.k_blocks; ++kb) {
          mbar_wait(bar_full + 8 * stage, phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kStageBytes);
          const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + kABytes);
          const uint32_t rem = args.I - kb * BK;
          const uint32_t nk = rem >= BK ? BK / 16 : (rem + 15) / 16;
          for (uint32_t kk = 0; kk < nk; ++kk)
            mma_bf16(d_tmem, da + 2 * kk, db + 2 * kk, idesc, (kb | kk) != 0);
          mma_commit(bar_empty + 8 * stage);
          if (++stage == kStages) stage = 0, phase ^= 1;
        }
        mma_commit(bar_tfull + 8 * buf);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------- epilogue
    const int e = warp - 4;            // 0..7
    const int q = warp & 3;            // TMEM lane quarter (warp % 4)
    const int half = e >> 2;           // column half: [half*128, half*128+128)
    const int row = q * 32 + lane;     // accumulator row == sample within tile
    const int et = threadIdx.x - 128;  // 0..255
    const uint32_t O = args.O;
    uint32_t i = 0;
    for (uint32_t t = t_begin; t < t_end; ++t, ++i) {
      const uint32_t m_tile = t % args.m_tiles, n_tile = t / args.m_tiles;
      const uint32_t buf = i & 1, use = (i >> 1) & 1;
      // stage this tile's per-spark b1 / W2^T / b2 (fp32) in shared memory
      epi_bar();
      for (int idx = et; idx < SPT * H; idx += kEpiThreads) {
        const int j = idx / H, h = idx % H;
        const uint64_t p = (uint64_t)n_tile * SPT + j;
        const bool ok = p < args.rows;
        const __nv_bfloat16* base = args.W + (ok ? p : 0) * args.Dp + (uint64_t)H * args.I;
        s_b1[idx] = ok ? __bfloat162float(base[h]) : 0.0f;
#pragma unroll
        for (int o = 0; o < kOPad; ++o)
          s_w2t[idx * kOPad + o] =
              (ok && (uint32_t)o < O) ? __bfloat162float(base[H + o * H + h]) : 0.0f;
      }
      for (int idx = et; idx < SPT * kOPad; idx += kEpiThreads) {
        const int j = idx / kOPad, o = idx % kOPad;
        const uint64_t p = (uint64_t)n_tile * SPT + j;
        float v = 0.0f;
        if (p < args.rows && (uint32_t)o < O)
          v = __bfloat162float(args.W[p * args.Dp + (uint64_t)H * args.I + H + (uint64_t)O * H + o]);
        s_b2[idx] = v;
      }
      const uint32_t s = m_tile * BM + row;
      const bool valid = s < args.S;
      const int label = valid ? args.y[s] : 0;
      epi_bar();

      mbar_wait(bar_tfull + 8 * buf, use);
      tc_fence_after();
      const uint32_t taddr = tmem_base + buf * BN + ((uint32_t)(q * 32) << 16);
      float z[kOPad];
#pragma unroll
      for (int o = 0; o < kOPad; ++o) z[o] = 0.0f;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int col0 = half * 128 + c * 32;
        float acc[32];
        tmem_ld32(taddr + col0, acc);
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int n = col0 + u;
          const float hv = fmaxf(acc[u] + s_b1[n], 0.0f);
          const float4* w = reinterpret_cast<const float4*>(s_w2t + n * kOPad);
          const float4 w0 = w[0], w1 = w[1], w2 = w[2];
          z[0] = fmaf(w0.x, hv, z[0]);
          z[1] = fmaf(w0.y, hv, z[1]);
          z[2] = fmaf(w0.z, hv, z[2]);
          z[3] = fmaf(w0.w, hv, z[3]);
          z[4] = fmaf(w1.x, hv, z[4]);
          z[5] = fmaf(w1.y, hv, z[5]);
          z[6] = fmaf(w1.z, hv, z[6]);
          z[7] = fmaf(w1.w, hv, z[7]);
          z[8] = fmaf(w2.x, hv, z[8]);
          z[9] = fmaf(w2.y, hv, z[9]);
          z[10] = fmaf(w2.z, hv, z[10]);
          z[11] = fmaf(w2.w, hv, z[11]);
        }
        if (!kSplitSpark && ((col0 + 32) % H) == 0) {
          const int j = col0 / H;  // spark within tile
          float loss = 0.0f;
          if (valid) {
            float zz[kOPad];
            float mx = -INFINITY;
#pragma unroll
            for (int o = 0; o < kOPad; ++o) {
              zz[o] = z[o] + s_b2[j * kOPad + o];
              if ((uint32_t)o < O) mx = fmaxf(mx, zz[o]);
            }
            float se = 0.0f, zl = 0.0f;
#pragma unroll
            for (int o = 0; o < kOPad; ++o) {
              if ((uint32_t)o < O) se += expf(zz[o] - mx);
              if (o == label) zl = zz[o];
            }
            loss = (mx + logf(se)) - zl;
          }
          loss = warp_sum(loss);
          if (lane == 0) s_red[e * 8 + (j - half * (SPT / 2))] = loss;
#pragma unroll
          for (int o = 0; o < kOPad; ++o) z[o] = 0.0f;
        }
      }
      // accumulator buffer consumed: hand it back to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_tempty + 8 * buf);

      if (kSplitSpark) {
        // H > 128: half 0 holds the partial logits of hidden [0,128)
        if (half == 0) {
#pragma unroll
          for (int o = 0; o < kOPad; ++o) s_z[row * kOPad + o] = z[o];
        }
        epi_bar();
        if (half == 1) {
          float loss = 0.0f;
          if (valid) {
            float zz[kOPad];
            float mx = -INFINITY;
#pragma unroll
            for (int o = 0; o < kOPad; ++o) {
              zz[o] = z[o] + s_z[row * kOPad + o] + s_b2[o];
              if ((uint32_t)o < O) mx = fmaxf(mx, zz[o]);
            }
            float se = 0.0f, zl = 0.0f;
#pragma unroll
            for (int o = 0; o < kOPad; ++o) {
              if ((uint32_t)o < O) se += expf(zz[o] - mx);
              if (o == label) zl = zz[o];
            }
            loss = (mx + logf(se)) - zl;
          }
          loss = warp_sum(loss);
          if (lane == 0) s_red[e * 8] = loss;
        }
      }
      epi_bar();
      // deterministic per-(spark, m-tile) partial: sum of the 4 lane quarters
      if (et < SPT) {
        const int j = et;
        const int h = kSplitSpark ? 1 : (j * H) / 128;
        const int jl = kSplitSpark ? 0 : j - h * (SPT / 2);
        float sum = 0.0f;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) sum += s_red[(h * 4 + qq) * 8 + jl];
        const uint64_t p = (uint64_t)n_tile * SPT + j;
        if (p < args.rows) {
          args.part[(p * args.m_tiles + m_tile) * 2] = sum;
          args.part[(p * args.m_tiles + m_tile) * 2 + 1] = 0.0f;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

// -------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

}  // namespace

template <int H>
static cudaError_t prepare_h();

struct MlpPlan {
  CUtensorMap tmap_x;
  CUtensorMap tmap_w;
  MlpArgs args;
  int grid;
  int H;
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
  if (O < 2 || O > (uint32_t)kMaxO - 2) return fail("MLP fitness: out_dim must be in [2, 10]");
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
  const uint32_t spt = BN / H;
  {
    cuuint64_t dims[3] = {I, H, rows};
    cuuint64_t strides[2] = {(cuuint64_t)I * 2, (cuuint64_t)Dp * 2};
    cuuint32_t box[3] = {BK, H, spt};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&p->tmap_w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<__nv_bfloat16*>(W), dims,
            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      delete p;
      return fail("MLP fitness: W tensor map encode failed");
    }
  }
  p->H = (int)H;
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
  const uint32_t tiles = p->args.m_tiles * p->args.n_tiles;
  p->grid = (int)(tiles < (uint32_t)nsm ? tiles : (uint32_t)nsm);
  cudaError_t e = H == 32    ? prepare_h<32>()
                  : H == 64  ? prepare_h<64>()
                  : H == 128 ? prepare_h<128>()
                             : prepare_h<256>();
  if (e != cudaSuccess) {
    delete p;
    return fail(cudaGetErrorString(e));
  }
  return p;
}

void mlp_plan_destroy(MlpPlan* p) { delete p; }

template <int H>
static cudaError_t launch_h(const MlpPlan* p, const MlpArgs& a, cudaStream_t s) {
  k_mlp_fitness<H><<<p->grid, kThreads, kSmemBytes, s>>>(p->tmap_x, p->tmap_w, a);
  return cudaGetLastError();
}

template <int H>
static cudaError_t prepare_h() {
  return cudaFuncSetAttribute(k_mlp_fitness<H>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kSmemBytes);
}

cudaError_t mlp_fitness_launch(const MlpPlan* p, float* part, const int* gate, cudaStream_t s) {
  MlpArgs a = p->args;
  a.part = part;
  a.gate = gate;
  switch (p->H) {
    case 32: return launch_h<32>(p, a, s);
    case 64: return launch_h<64>(p, a, s);
    case 128: return launch_h<128>(p, a, s);
    case 256: return launch_h<256>(p, a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace mgfwa_b200
