// k_lenet.cu — LeNet-5 loss of every candidate (SURVEY.md §8(a) a10, config
// C3): conv5x5 1->6 (pad 2) -> ReLU -> avgpool2 -> conv5x5 6->16 -> ReLU ->
// avgpool2 -> fc 400->120 -> ReLU -> fc 120->84 -> ReLU -> fc 84->10 -> CE,
// mean over the S synthetic samples.  Parameter layout and arithmetic follow
// the fp64 restatement oracle/mgfwa_oracle.c f_lenet (PyTorch Conv2d/Linear
// weight order: c1w[6][1][5][5], c1b, c2w[16][6][5][5], c2b, f1w[120][400],
// f1b, f2w[84][120], f2b, f3w[10][84], f3b).
//
// Every candidate has its own weights, so the convolutions are per-candidate
// implicit GEMMs with N = 6 (conv1) and N = 16 (conv2) output channels: far
// below tcgen05's 128-row MMA tile, and each candidate's conv2 A operand
// (pooled conv1 activations) is produced on chip.  They run on the warp-level
// tensor-core MMA (mma.sync m16n8k16 bf16 -> fp32) in two kernels per
// evaluation:
//
// k_lenet_conv — one sample per warp, 12 warps per SM, no block-wide
// synchronisation inside a work item (candidate x 128-sample chunk); only the
// candidate's conv weights are staged (B fragments then live in registers):
//   * conv1: M = 784 output pixels as 25 tile pairs (conv1_pairs): a pair =
//     8 pool windows (MMA row g), its two tiles the windows' two pixel rows,
//     MMA rows g / g + 8 their two columns, so a thread holds all four pixels
//     of its window (ReLU + pool in registers, no shuffle); K = 5 rows x 6
//     taps (kx padded), A fragments read from the sample's "pair image"
//     (x, x+1) — each register pair one 64-bit load — precomputed once per
//     plan (the dataset never changes) and prefetched with cp.async
//     (conv1_tiles, the single-tile form with a shuffle, is kept behind
//     LENET_CONV1_PAIRS=0 and gives bit-identical results);
//   * conv2: M = 100 pixels in pool order (rows r / r + 8 a window's two pixel
//     rows, the horizontal pair one shuffle), K = 25 taps x 8 channels (6 + 2
//     zero), N = 16, taps ordered so that a fragment's row-(g+8) word equals
//     its second tap's row-g word (conv2_k): 30 shared-memory loads per tile
//     feed 26 MMAs;
//   * the pooled output ([window][16 channels] bf16, 800 B per sample) goes to
//     a scratch buffer in HBM (at most kScratchBytes; candidates are processed
//     in groups that fit).
// k_lenet_fc — one work item = (candidate, 128-sample chunk): fc1 (M = 128
//   outputs: one 16-row tile per warp, whose A fragments stay in registers for
//   all the candidate's chunks) x N = 128 samples, fc2 and fc3 with B via
//   ldmatrix from the chunk's activations, CE per sample, fixed-order sums.
// Activations between layers are bf16, accumulation fp32, CE in fp32.
// Output: part[(row * nparts + p) * 2] = sum of CE over sample chunk p (128
// samples), slot 1 = 0 — the same partial-sum contract as k_mlp_fitness.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "common.cuh"
#include "kernels.h"
#include "tc_glue.cuh"

namespace mgfwa_b200 {

namespace {

constexpr uint32_t kChunkS = 128;  // samples per work item (one partial)

// parameter offsets in the candidate row (oracle f_lenet)
constexpr int oC1W = 0, oC1B = 150, oC2W = 156, oC2B = 2556, oF1W = 2572, oF1B = 50572,
              oF2W = 50692, oF2B = 60772, oF3W = 60856, oF3B = 61696;
constexpr int kLenetDim = 61706;

// shared-memory layout (bytes); strides chosen for conflict-free fragment
// loads (32-bit) and 16-byte aligned ldmatrix rows.
constexpr int kC1K = 32;    // conv1 K: 5 rows x 6 taps + 2 pad
constexpr int kC2S = 216;   // conv2 weight row stride (bf16), K = 25 taps x 8 + 8 pad
#ifndef LENET_CONV1_PAIRS
#define LENET_CONV1_PAIRS 1  // conv1 on tile pairs (whole pool windows per thread, 64-bit loads)
#endif
#ifndef LENET_CV_P1T
#define LENET_CV_P1T 4  // conv1 tile pairs in flight per warp (measured: 4 < 3 < 5)
#endif
// pair-image row stride (32-bit words, 33 rows): tile pairs load 64-bit words and
// are conflict-light at 8 mod 32; single tiles load 32-bit words, conflict-free at 4 mod 32
constexpr int kImgS = LENET_CONV1_PAIRS ? 40 : 36;
constexpr int kImgWords = 33 * kImgS;  // 1188 words (16-byte multiple)
constexpr int kP1R = 21;    // pooled conv1 map row stride (pixels; = 1 mod 4, 4 kP1R = 20 mod 32), 14 rows x 4 words
constexpr int kP1Words = 14 * kP1R * 4;

struct LenetArgs {
  const uint32_t* pimg;    // [S][1092] pair images of the samples
  const int32_t* y;        // [S]
  const __nv_bfloat16* W;  // [rows][Dp]
  uint64_t rows, Dp;
  uint32_t S, nparts;
  float* part;
  const int* gate;
};

__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 t = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&t);
}

__device__ __forceinline__ float bf(const __nv_bfloat16 x) { return __bfloat162float(x); }

// conv1 K order.  Pair q = 8 st + 4 h + c (the A-fragment k pair 2c[+8] of
// k16-step st held by lane quad c) covers taps (ky, 2 kxp) and (ky, 2 kxp + 1):
// q < 12: ky = c, kxp = q / 4; q = 12..14: ky = 4, kxp = c; q = 15: padding.
// A conv1 tile is a 2 x 2 block of pool windows; with the pair image's row
// stride = 4 mod 32 the 32 words of every A-fragment load fall in distinct
// banks (checked exhaustively over the 49 tiles and 8 loads).
__host__ __device__ constexpr int conv1_k(int ky, int kx) {
  return ky < 4 ? 2 * (4 * (kx >> 1) + ky) + (kx & 1) : 2 * (12 + (kx >> 1)) + (kx & 1);
}


// Prefetch one sample's pair image into this warp's buffer (cp.async).
__device__ __forceinline__ void prefetch_img(uint32_t dst, const uint32_t* src, int lane) {
  for (int i = lane; i < kImgWords / 4; i += 32) cp_async16(dst + 16 * i, src + 4 * i);
  cp_async_commit();
}

}  // namespace

// Pair images of the dataset: P[s][Y][X] = (x[s][Y-2][X-2], x[s][Y-2][X-1]),
// zero outside the 28 x 28 image, 33 rows x kImgS words.
__global__ void k_lenet_pairs(const __nv_bfloat16* X, uint32_t S, uint32_t* P) {
  const uint64_t n = (uint64_t)S * kImgWords;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = i / kImgWords;
    const int r = (int)(i % kImgWords), Y = r / kImgS, Xc = r % kImgS;
    const int yy = Y - 2, x0 = Xc - 2, x1 = Xc - 1;
    const bool iny = yy >= 0 && yy < 28;
    const __nv_bfloat16* img = X + s * 784;
    __nv_bfloat162 pr;
    pr.x = (iny && x0 >= 0 && x0 < 28) ? img[yy * 28 + x0] : __float2bfloat16(0.0f);
    pr.y = (iny && x1 >= 0 && x1 < 28) ? img[yy * 28 + x1] : __float2bfloat16(0.0f);
    P[i] = *reinterpret_cast<uint32_t*>(&pr);
  }
}

namespace {

#ifndef LENET_CV_WARPS
#define LENET_CV_WARPS 12
#endif
#ifndef LENET_CV_C1T
#define LENET_CV_C1T 7
#endif
#ifndef LENET_CV_C2T
#define LENET_CV_C2T 2
#endif
constexpr int kConvWarps = LENET_CV_WARPS;
constexpr int kCvC1T = LENET_CV_C1T;  // conv1 tiles in flight per warp
constexpr int kCvC2T = LENET_CV_C2T;  // conv2 tiles in flight per warp (x 2 n-tiles)
constexpr int kConvThreads = kConvWarps * 32;
constexpr int kP2Row = 416;  // bf16 per sample in the scratch: K' = ch * 25 + window + 4 (kF1Shift), zero pads
constexpr uint64_t kScratchBytes = 2ull << 30;  // activation scratch cap (C3: 1.23 GB)

struct ConvSmem {
  static constexpr int wc1 = 0;                                // [8][32] bf16
  static constexpr int wc2 = wc1 + 8 * kC1K * 2;               // [16][216] bf16
  static constexpr int bc1 = wc2 + 16 * kC2S * 2;              // f32 [8]
  static constexpr int bc2 = bc1 + 8 * 4;                      // f32 [16]
  static constexpr int img = bc2 + 16 * 4;                     // per warp [33][40] u32
  static constexpr int p1 = img + kConvWarps * kImgWords * 4;  // per warp [14][kP1R][4] u32
  static constexpr int p2 = p1 + kConvWarps * kP1Words * 4;    // per warp [416] bf16 (K' row)
  static constexpr int total = p2 + kConvWarps * kP2Row * 2;
};
static_assert(ConvSmem::img % 16 == 0 && ConvSmem::p2 % 16 == 0, "aligned cp.async / uint4 regions");

struct LenetSplitArgs {
  LenetArgs base;
  uint64_t row0;      // first candidate of the group (tensor-map row coordinate)
  __nv_bfloat16* p2;  // [rows][S][416] scratch (K' rows)
};

}  // namespace

// conv1 on tiles t0 .. t0 + N - 1 (4 pool windows each) of one sample:
// ReLU + 2x2 average pool -> p1[window][channel pair] (bf16 pairs).
template <int N>
__device__ __forceinline__ void conv1_tiles(int t0, const uint32_t* imgc, const uint32_t* imgd, uint32_t* p1,
                                            int wi, int dx, int c, const uint32_t (&bw1)[2][2], float b1a,
                                            float b1b) {
  int wpos[N];
  float d[N][4];
#pragma unroll
  for (int u = 0; u < N; ++u) {
    const int ty = (t0 + u) / 7, tx = (t0 + u) - 7 * ty;  // tile = windows 2ty..+1 x 2tx..+1
    const int py = 2 * ty + (wi >> 1), px = 2 * tx + (wi & 1);
    wpos[u] = py * kP1R + px;
    const int base0 = (2 * py) * kImgS + 2 * px + dx, base1 = base0 + kImgS;
    d[u][0] = b1a, d[u][1] = b1b, d[u][2] = b1a, d[u][3] = b1b;
    mma_bf16(d[u], imgc[base0], imgc[base1], imgc[base0 + 2], imgc[base1 + 2], bw1[0][0], bw1[0][1]);
    mma_bf16(d[u], imgc[base0 + 4], imgc[base1 + 4], imgd[base0], imgd[base1], bw1[1][0], bw1[1][1]);
  }
#pragma unroll
  for (int u = 0; u < N; ++u) {
    // ReLU, vertical pair in-thread (rows g, g+8), horizontal pair = lane ^ 4
    float s0 = fmaxf(d[u][0], 0.f) + fmaxf(d[u][2], 0.f);
    float s1 = fmaxf(d[u][1], 0.f) + fmaxf(d[u][3], 0.f);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 4);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 4);
    if (dx == 0) p1[wpos[u] * 4 + c] = pack_bf16(s0, s1);
  }
}

// conv1 on tile pairs t0 .. t0 + N - 1 of one sample (25 pairs): pair t
// covers pool windows 8t .. 8t + 7 (row g of the MMA tile = window 8t + g),
// tile dy of the pair the window's pixel row dy, and MMA rows g / g + 8 its
// columns dx = 0 / 1.  A thread then holds all four pixels of its window for
// its two channels: ReLU + 2x2 pool in registers (same summation order as
// conv1_tiles: (p00 + p10) + (p01 + p11), so p1 is bit-identical), no
// shuffle, every lane stores, and each A-fragment register pair (rows g, g+8
// = neighbouring pair-image words) is one 64-bit load.
template <int N>
__device__ __forceinline__ void conv1_pairs(int t0, const uint32_t* imgc, const uint32_t* imgd, uint32_t* p1, int g,
                                            int c, const uint32_t (&bw1)[2][2], float b1a, float b1b) {
  int wpos[N];
  float d[N][2][4];
#pragma unroll
  for (int u = 0; u < N; ++u) {
    const int w0 = 8 * (t0 + u) + g;
    const int w = w0 < 196 ? w0 : 195;  // the last pair's 4 spare rows recompute window 195
    const int py = w / 14, px = w - 14 * py;
    wpos[u] = w0 < 196 ? py * kP1R + px : -1;
    const int X = (2 * py) * kImgS + 2 * px;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const uint2 a01 = *reinterpret_cast<const uint2*>(imgc + X + dy * kImgS);      // kxp 0, dx 0 / 1
      const uint2 a23 = *reinterpret_cast<const uint2*>(imgc + X + dy * kImgS + 2);  // kxp 1
      const uint2 e01 = *reinterpret_cast<const uint2*>(imgc + X + dy * kImgS + 4);  // kxp 2
      const uint2 e23 = *reinterpret_cast<const uint2*>(imgd + X + dy * kImgS);      // ky 4
      d[u][dy][0] = b1a, d[u][dy][1] = b1b, d[u][dy][2] = b1a, d[u][dy][3] = b1b;
      mma_bf16(d[u][dy], a01.x, a01.y, a23.x, a23.y, bw1[0][0], bw1[0][1]);
      mma_bf16(d[u][dy], e01.x, e01.y, e23.x, e23.y, bw1[1][0], bw1[1][1]);
    }
  }
#pragma unroll
  for (int u = 0; u < N; ++u) {
    const float s0 = (fmaxf(d[u][0][0], 0.f) + fmaxf(d[u][1][0], 0.f)) + (fmaxf(d[u][0][2], 0.f) + fmaxf(d[u][1][2], 0.f));
    const float s1 = (fmaxf(d[u][0][1], 0.f) + fmaxf(d[u][1][1], 0.f)) + (fmaxf(d[u][0][3], 0.f) + fmaxf(d[u][1][3], 0.f));
    if (wpos[u] >= 0) p1[wpos[u] * 4 + c] = pack_bf16(s0, s1);
  }
}

// conv2 K order for the column-reuse scheme (k_lenet_conv): k-step st holds
// two taps A (k 0-7) and B (k 8-15), 8 channels each (6 + 2 zero).
//   st = 2 kx + h (kx < 5, h < 2): A = (2h, kx), B = (2h + 1, kx)
//   st = 10 + j (j < 3):           A = (4, 2j), B = (4, 2j + 1)   [(4, 5) = zero padding]
// In the MMA fragment a lane's rows g and g + 8 are vertically adjacent
// pixels, so a1 (row g + 8, tap A) is the same word as a2 (row g, tap B =
// tap A one row down): per pool tile and kernel column the lane loads the 6
// words of rows 0..5 once and feeds 2-3 MMAs from them — 30 shared-memory
// loads per tile instead of 52.
__host__ __device__ constexpr int conv2_k(int ky, int kx) {
  return ky < 4 ? 16 * (2 * kx + (ky >> 1)) + 8 * (ky & 1) : 16 * (10 + (kx >> 1)) + 8 * (kx & 1);
}

// The pooled conv2 output of the sample in fc1's K order K' = ch * 25 +
// window + 4 (kF1Shift).  IL = false: o = the sample's K' row (scratch path,
// k_lenet_conv -> k_lenet_fc_tc).  IL = true: o = the sample's row base inside
// the fc1 A operand of the fused kernel (tcgen05 no-swizzle K-major layout,
// K' chunk stride 2048 bytes).
template <int N, bool IL>
__device__ __forceinline__ void conv2_tiles(int t0, const uint32_t* p1c, __nv_bfloat16* o, int wi, int dx,
                                            int c, const uint32_t (&bw2)[13][2][2], float b2a, float b2b,
                                            float b2c, float b2d) {
  int wv[N];
  const uint32_t* q[N];
  float d[N][2][4];
#pragma unroll
  for (int u = 0; u < N; ++u) {
    const int w = 4 * (t0 + u) + wi;
    wv[u] = w < 25 ? w : -1;
    // window 4t + wi has (qy + qx) = wi mod 4 and the map's row stride is 1 mod
    // 4 pixels, so the 8 pixels of a tile row hit distinct bank quads; the
    // padding slots of the last tile repeat its window 24 (same words)
    const int wc = w < 25 ? w : 24;
    const int qy = wc / 5, qx = wc - 5 * qy;
    q[u] = p1c + ((2 * qy) * kP1R + 2 * qx + dx) * 4;
    d[u][0][0] = b2a, d[u][0][1] = b2b, d[u][0][2] = b2a, d[u][0][3] = b2b;
    d[u][1][0] = b2c, d[u][1][1] = b2d, d[u][1][2] = b2c, d[u][1][3] = b2d;
  }
  uint32_t r4p[N], r5p[N];
#pragma unroll
  for (int kx = 0; kx < 5; ++kx) {
    uint32_t r[N][6];
#pragma unroll
    for (int u = 0; u < N; ++u)
#pragma unroll
      for (int j = 0; j < 6; ++j) r[u][j] = q[u][(j * kP1R + kx) * 4];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int u = 0; u < N; ++u)
#pragma unroll
        for (int n = 0; n < 2; ++n)
          mma_bf16(d[u][n], r[u][2 * h], r[u][2 * h + 1], r[u][2 * h + 1], r[u][2 * h + 2],
                   bw2[2 * kx + h][n][0], bw2[2 * kx + h][n][1]);
    if (kx & 1) {
#pragma unroll
      for (int u = 0; u < N; ++u)
#pragma unroll
        for (int n = 0; n < 2; ++n)
          mma_bf16(d[u][n], r4p[u], r5p[u], r[u][4], r[u][5], bw2[10 + kx / 2][n][0], bw2[10 + kx / 2][n][1]);
    } else if (kx == 4) {
#pragma unroll
      for (int u = 0; u < N; ++u)
#pragma unroll
        for (int n = 0; n < 2; ++n)
          mma_bf16(d[u][n], r[u][4], r[u][5], 0u, 0u, bw2[12][n][0], bw2[12][n][1]);
    }
#pragma unroll
    for (int u = 0; u < N; ++u) r4p[u] = r[u][4], r5p[u] = r[u][5];
  }
#pragma unroll
  for (int u = 0; u < N; ++u) {
    float s0 = fmaxf(d[u][0][0], 0.f) + fmaxf(d[u][0][2], 0.f);
    float s1 = fmaxf(d[u][0][1], 0.f) + fmaxf(d[u][0][3], 0.f);
    float s2 = fmaxf(d[u][1][0], 0.f) + fmaxf(d[u][1][2], 0.f);
    float s3 = fmaxf(d[u][1][1], 0.f) + fmaxf(d[u][1][3], 0.f);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 4);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 4);
    s2 += __shfl_xor_sync(0xffffffffu, s2, 4);
    s3 += __shfl_xor_sync(0xffffffffu, s3, 4);
    if (dx == 0 && wv[u] >= 0) {
      const int w = wv[u];
      const float vals[4] = {s0, s1, s2, s3};
      const int chs[4] = {2 * c, 2 * c + 1, 8 + 2 * c, 9 + 2 * c};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = chs[q] * 25 + w + 4;
        o[IL ? (k >> 3) * 1024 + (k & 7) : k] = __float2bfloat16(vals[q]);
      }
    }
  }
}

__global__ void __launch_bounds__(kConvThreads, 1) k_lenet_conv(LenetSplitArgs sa) {
  pdl_enter();
  const LenetArgs& args = sa.base;
  if (args.gate != nullptr && *args.gate == 0) return;
  extern __shared__ __align__(16) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int wi = g >> 1, dx = g & 1;
  __nv_bfloat16* wc1 = reinterpret_cast<__nv_bfloat16*>(sm + ConvSmem::wc1);
  __nv_bfloat16* wc2 = reinterpret_cast<__nv_bfloat16*>(sm + ConvSmem::wc2);
  float* bc1 = reinterpret_cast<float*>(sm + ConvSmem::bc1);
  float* bc2 = reinterpret_cast<float*>(sm + ConvSmem::bc2);
  const uint32_t* img = reinterpret_cast<const uint32_t*>(sm + ConvSmem::img) + warp * kImgWords;
  const uint32_t img_s = smem_addr(img);
  uint32_t* p1 = reinterpret_cast<uint32_t*>(sm + ConvSmem::p1) + warp * kP1Words;
  __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(sm + ConvSmem::p2) + warp * kP2Row;
  {
    uint32_t* p = reinterpret_cast<uint32_t*>(sm);
    for (int i = threadIdx.x; i < ConvSmem::total / 4; i += kConvThreads) p[i] = 0u;
  }
  __syncthreads();
  const uint32_t* imgc = img + c * kImgS;
  const uint32_t* imgd = img + 4 * kImgS + 2 * (c < 3 ? c : 2);
  const uint32_t* p1c = p1 + c;

  const uint64_t total = args.rows * args.nparts;
  const uint64_t t_begin = total * blockIdx.x / gridDim.x;
  const uint64_t t_end = total * (blockIdx.x + 1) / gridDim.x;
  uint64_t staged = ~0ull;
  uint32_t bw1[2][2], bw2[13][2][2];
  float b1a = 0.f, b1b = 0.f, b2a = 0.f, b2b = 0.f, b2c = 0.f, b2d = 0.f;
  for (uint64_t item = t_begin; item < t_end; ++item) {
    const uint64_t row = item / args.nparts;
    const uint32_t part = (uint32_t)(item % args.nparts);
    const uint32_t s_lo = part * kChunkS, s_hi = min(args.S, s_lo + kChunkS);
    if (row != staged) {
      __syncthreads();
      // conv weights and biases pre-scaled by 1/4 (exact): the 2 x 2 average
      // pools then reduce to sums of ReLUs, relu(x) / 4 = relu(x / 4)
      const __nv_bfloat16* w = args.W + row * args.Dp;
      for (int i = threadIdx.x; i < 150; i += kConvThreads) {
        const int ch = i / 25, r = i % 25, ky = r / 5, kx = r % 5;
        wc1[ch * kC1K + conv1_k(ky, kx)] = __float2bfloat16(0.25f * bf(w[oC1W + i]));
      }
      for (int i = threadIdx.x; i < 2400; i += kConvThreads) {
        const int ch = i / 150, r = i % 150, ci = r / 25, tap = r % 25;
        wc2[ch * kC2S + conv2_k(tap / 5, tap % 5) + ci] = __float2bfloat16(0.25f * bf(w[oC2W + i]));
      }
      if (threadIdx.x < 6) bc1[threadIdx.x] = 0.25f * bf(w[oC1B + threadIdx.x]);
      if (threadIdx.x < 16) bc2[threadIdx.x] = 0.25f * bf(w[oC2B + threadIdx.x]);
      __syncthreads();
      staged = row;
#pragma unroll
      for (int st = 0; st < 2; ++st) {
        const __nv_bfloat16* b = wc1 + g * kC1K + 16 * st + 2 * c;
        bw1[st][0] = *reinterpret_cast<const uint32_t*>(b);
        bw1[st][1] = *reinterpret_cast<const uint32_t*>(b + 8);
      }
#pragma unroll
      for (int st = 0; st < 13; ++st)
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          const __nv_bfloat16* b = wc2 + (8 * n + g) * kC2S + 16 * st + 2 * c;
          bw2[st][n][0] = *reinterpret_cast<const uint32_t*>(b);
          bw2[st][n][1] = *reinterpret_cast<const uint32_t*>(b + 8);
        }
      b1a = bc1[2 * c], b1b = bc1[2 * c + 1];
      b2a = bc2[2 * c], b2b = bc2[2 * c + 1], b2c = bc2[8 + 2 * c], b2d = bc2[9 + 2 * c];
    }
    if (s_lo + warp < s_hi) prefetch_img(img_s, args.pimg + (uint64_t)(s_lo + warp) * kImgWords, lane);
    for (uint32_t s = s_lo + warp; s < s_hi; s += kConvWarps) {
      cp_async_wait_all();
      __syncwarp();
      // ---- conv1 + ReLU + pool -> p1: 49 tiles
#if LENET_CONV1_PAIRS
#pragma unroll 1
      for (int t0 = 0; t0 + LENET_CV_P1T <= 25; t0 += LENET_CV_P1T)
        conv1_pairs<LENET_CV_P1T>(t0, imgc, imgd, p1, g, c, bw1, b1a, b1b);
      if constexpr (25 % LENET_CV_P1T != 0)
        conv1_pairs<25 % LENET_CV_P1T>(25 - 25 % LENET_CV_P1T, imgc, imgd, p1, g, c, bw1, b1a, b1b);
#else
#pragma unroll 1
      for (int t0 = 0; t0 + kCvC1T <= 49; t0 += kCvC1T)
        conv1_tiles<kCvC1T>(t0, imgc, imgd, p1, wi, dx, c, bw1, b1a, b1b);
      if constexpr (49 % kCvC1T != 0) conv1_tiles<49 % kCvC1T>(49 - 49 % kCvC1T, imgc, imgd, p1, wi, dx, c, bw1, b1a, b1b);
#endif
      __syncwarp();
      if (s + kConvWarps < s_hi)
        prefetch_img(img_s, args.pimg + (uint64_t)(s + kConvWarps) * kImgWords, lane);
      // ---- conv2 + ReLU + pool -> o (the K' row): 7 tiles
#pragma unroll 1
      for (int t0 = 0; t0 + kCvC2T <= 7; t0 += kCvC2T)
        conv2_tiles<kCvC2T, false>(t0, p1c, o, wi, dx, c, bw2, b2a, b2b, b2c, b2d);
      if constexpr (7 % kCvC2T != 0)
        conv2_tiles<7 % kCvC2T, false>(7 - 7 % kCvC2T, p1c, o, wi, dx, c, bw2, b2a, b2b, b2c, b2d);
      __syncwarp();
      // ---- p2 row -> scratch (832 B, coalesced 16-byte stores)
      uint4* dst = reinterpret_cast<uint4*>(sa.p2 + (row * args.S + s) * (uint64_t)kP2Row);
      const uint4* srcv = reinterpret_cast<const uint4*>(o);
      for (int i = lane; i < kP2Row * 2 / 16; i += 32) dst[i] = srcv[i];
      __syncwarp();
    }
  }
}

// ============================================================ fc on tcgen05
// The fc stack of a work item (candidate, 128-sample chunk) on the 5th-gen
// tensor cores, shared by k_lenet_fc_tc (split path: pooled conv2 rows from
// the HBM scratch) and k_lenet_fused (rows produced in shared memory):
//   fc1 = tcgen05.mma kind::f16, M = 128 samples, N = 128 (120 outputs),
//         K' = 416 (K = 400 shifted by kF1Shift), A (pooled conv2 rows) and
//         B (f1w, two TMA-loaded K' halves) in shared memory, D1 in TMEM;
//   fc2 / fc3: +b, ReLU, bf16 -> back into TMEM (tcgen05.st) as the A
//         operand (M = 128, N = 96 (84) / 16 (10), K = 128 (120) / 96 (84),
//         B = f2w / f3w in shared memory);
//   logits (tcgen05.ld, one sample per thread) -> CE -> fixed-order sums.
// TMEM columns: A2 [0, 64), A3 [64, 112), D1 [256, 384), D2 [384, 480),
// D3 [480, 496) of a 512-column allocation.
//
// fc1's K index is shifted by kF1Shift = 4 (K' = channel * 25 + window + 4;
// A is zero outside [4, 404)): f1w starts 8 bytes off a 16-byte boundary in
// the candidate row, and with the shift every 16-byte K' chunk of it is
// 16-byte aligned in global memory, as TMA requires.  tmap_f1 = 3-D view
// (K', j, candidate) of every candidate's f1w block based 4 parameters before
// it; a box (8, 128, 1) is one 16-byte K' chunk of the 128 (120 + 8
// zero-filled) rows, which lands in shared memory as one 2048-byte column of
// core matrices of the no-swizzle K-major operand layout.  K' in [0, 4) reads
// the 4 parameters before f1w (c2b), which meet zeros in A; K' >= 404 is
// zero-filled.
namespace {

constexpr int kF1Shift = 4;
constexpr int kF1K = 416;                     // K' (26 MMA k-steps)
constexpr int kF1Half = 208;                  // K' per f1w half (13 k-steps)
constexpr int kA1Bytes = 128 * kF1K * 2;      // fc1 A: 128 rows x 416
constexpr int kW1HalfBytes = 128 * kF1Half * 2;
static_assert(kF1Shift == 4 && kP2Row == kF1K, "scratch rows are fc1 A rows");
constexpr uint32_t kColA2 = 0, kColA3 = 64, kColD1 = 256, kColD2 = 384, kColD3 = 480;
constexpr int kFcThreadsTc = 256;  // 8 warps: TMEM lane quarter = warp % 4, column half = warp / 4

// byte offset of element (r, k) in a no-swizzle K-major tcgen05 operand of
// R rows: 8-row x 16-byte core matrices, LBO (along K) = R * 16, SBO = 128
__host__ __device__ constexpr uint32_t il_off(uint32_t r, uint32_t k, uint32_t R) {
  return (k >> 3) * (R * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

// fc2 / fc3 operands and the biases (staged once per candidate)
struct FcTail {
  static constexpr int w2 = 0;                  // fc2 B: 96 x 128 bf16
  static constexpr int w3 = w2 + 96 * 128 * 2;  // fc3 B: 16 x 96 bf16
  static constexpr int b1 = w3 + 16 * 96 * 2;   // f32 [128]
  static constexpr int b2 = b1 + 128 * 4;       // f32 [96]
  static constexpr int b3 = b2 + 96 * 4;        // f32 [16]
  static constexpr int red = b3 + 16 * 4;       // f32 [4]
  static constexpr int bytes = red + 16;
};

// 16 bytes = parameters [k0, k0 + 8) of a row (8-byte aligned source), 0 past `kmax`
__device__ __forceinline__ uint4 load8(const __nv_bfloat16* rowp, int k0, int kmax) {
  if (k0 + 8 <= kmax) {
    const uint2 a = *reinterpret_cast<const uint2*>(rowp + k0);
    const uint2 b = *reinterpret_cast<const uint2*>(rowp + k0 + 4);
    return make_uint4(a.x, a.y, b.x, b.y);
  }
  uint16_t v[8];
  const uint16_t* r = reinterpret_cast<const uint16_t*>(rowp);
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = k0 + q < kmax ? r[k0 + q] : (uint16_t)0;
  return make_uint4(v[0] | (uint32_t)v[1] << 16, v[2] | (uint32_t)v[3] << 16, v[4] | (uint32_t)v[5] << 16,
                    v[6] | (uint32_t)v[7] << 16);
}

__device__ __forceinline__ void async_smem_fence() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// f2w / f3w (rows past 84 / 10 and K past 120 / 84 zero) and the fc biases of
// candidate row w (all threads of the block; the caller synchronises)
__device__ __forceinline__ void stage_fc_tail(uint8_t* t, const __nv_bfloat16* w, int nthreads) {
  for (int i = threadIdx.x; i < 96 * 16; i += nthreads) {
    const int j = i / 16, cc = i - 16 * j;
    const uint4 v = j < 84 ? load8(w + oF2W + j * 120, 8 * cc, 120) : make_uint4(0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(t + FcTail::w2 + il_off(j, 8 * cc, 96)) = v;
  }
  for (int i = threadIdx.x; i < 16 * 12; i += nthreads) {
    const int j = i / 12, cc = i - 12 * j;
    const uint4 v = j < 10 ? load8(w + oF3W + j * 84, 8 * cc, 84) : make_uint4(0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(t + FcTail::w3 + il_off(j, 8 * cc, 16)) = v;
  }
  float* b1 = reinterpret_cast<float*>(t + FcTail::b1);
  float* b2 = reinterpret_cast<float*>(t + FcTail::b2);
  float* b3 = reinterpret_cast<float*>(t + FcTail::b3);
  for (int i = threadIdx.x; i < 128; i += nthreads) {
    b1[i] = i < 120 ? bf(w[oF1B + i]) : 0.f;
    if (i < 96) b2[i] = i < 84 ? bf(w[oF2B + i]) : 0.f;
    if (i < 16) b3[i] = i < 10 ? bf(w[oF3B + i]) : 0.f;
  }
  async_smem_fence();  // f2w / f3w are read by the tensor core
}

// One MMA round: issued by thread 0, every thread waits for its commit.
struct MmaBar {
  uint32_t bar, phase;
  __device__ __forceinline__ void wait() {
    tc::mbar_wait(bar, phase);
    phase ^= 1;
    tc::tc_fence_after();
  }
};

// fc1 k-steps [kk0, kk1) (A chunk 2 kk of a1_s, B chunk 2 (kk - kb) of w1_s)
__device__ __forceinline__ void fc1_mma(uint32_t tmem, uint32_t a1_s, uint32_t w1_s, int kk0, int kk1, int kb,
                                        uint32_t bar) {
  using namespace tc;
  tc_fence_after();
  constexpr uint32_t id1 = idesc_bf16(128, 128);
  for (int kk = kk0; kk < kk1; ++kk)
    mma_ss(tmem + kColD1, interleaved_desc(a1_s + kk * 2 * 2048, 2048, 128),
           interleaved_desc(w1_s + (kk - kb) * 2 * 2048, 2048, 128), id1, kk != 0);
  mma_commit(bar);
}

// After fc1's MMAs: fc1 epilogue -> A2, fc2, epilogue -> A3, fc3, CE over
// the chunk's samples [s_lo, s_hi); thread 0 returns the chunk's loss sum
// (fixed order: lanes, then the 4 lane quarters).  All threads of the
// 256-thread block call it.
__device__ float fc_tail(uint32_t tmem, const uint8_t* t, MmaBar& mb, uint32_t s_lo, uint32_t s_hi,
                         const int32_t* y) {
  using namespace tc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, hf = warp >> 2;
  const uint32_t lanes = tmem + ((uint32_t)(q * 32) << 16);
  const float* sb1 = reinterpret_cast<const float*>(t + FcTail::b1);
  const float* sb2 = reinterpret_cast<const float*>(t + FcTail::b2);
  const float* sb3 = reinterpret_cast<const float*>(t + FcTail::b3);
  float* red = const_cast<float*>(reinterpret_cast<const float*>(t + FcTail::red));
  const uint32_t w2_s = smem_addr(t + FcTail::w2), w3_s = smem_addr(t + FcTail::w3);
#pragma unroll 1
  for (int cc = 0; cc < 2; ++cc) {  // D1 columns [hf * 64, + 64)
    const int col0 = hf * 64 + cc * 32;
    float acc[32];
    tmem_ld32(lanes + kColD1 + col0, acc);
    uint32_t pk[16];
#pragma unroll
    for (int u = 0; u < 16; ++u)
      pk[u] = pack_bf16(fmaxf(acc[2 * u] + sb1[col0 + 2 * u], 0.f), fmaxf(acc[2 * u + 1] + sb1[col0 + 2 * u + 1], 0.f));
    tmem_st16(lanes + kColA2 + col0 / 2, pk);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc_fence_after();
    constexpr uint32_t id2 = idesc_bf16(128, 96);
    for (int kk = 0; kk < 8; ++kk)
      mma_ts(tmem + kColD2, tmem + kColA2 + 8 * kk, interleaved_desc(w2_s + kk * 2 * 1536, 1536, 128), id2, kk != 0);
    mma_commit(mb.bar);
  }
  mb.wait();
  {  // D2 columns [hf * 48, + 48) = 32 + 16
    const int col0 = hf * 48;
    float acc[32];
    tmem_ld32(lanes + kColD2 + col0, acc);
    uint32_t pk[16];
#pragma unroll
    for (int u = 0; u < 16; ++u)
      pk[u] = pack_bf16(fmaxf(acc[2 * u] + sb2[col0 + 2 * u], 0.f), fmaxf(acc[2 * u + 1] + sb2[col0 + 2 * u + 1], 0.f));
    tmem_st16(lanes + kColA3 + col0 / 2, pk);
    float acc2[16];
    tmem_ld16(lanes + kColD2 + col0 + 32, acc2);
    uint32_t pk2[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      pk2[u] = pack_bf16(fmaxf(acc2[2 * u] + sb2[col0 + 32 + 2 * u], 0.f),
                         fmaxf(acc2[2 * u + 1] + sb2[col0 + 32 + 2 * u + 1], 0.f));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     lanes + kColA3 + (col0 + 32) / 2),
                 "r"(pk2[0]), "r"(pk2[1]), "r"(pk2[2]), "r"(pk2[3]), "r"(pk2[4]), "r"(pk2[5]), "r"(pk2[6]),
                 "r"(pk2[7])
                 : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc_fence_after();
    constexpr uint32_t id3 = idesc_bf16(128, 16);
    for (int kk = 0; kk < 6; ++kk)
      mma_ts(tmem + kColD3, tmem + kColA3 + 8 * kk, interleaved_desc(w3_s + kk * 2 * 256, 256, 128), id3, kk != 0);
    mma_commit(mb.bar);
  }
  mb.wait();
  if (hf == 0) {  // logits: one sample per thread
    float z[16];
    tmem_ld16(lanes + kColD3, z);
    float loss = 0.f;
    const uint32_t smp = s_lo + q * 32 + lane;
    if (smp < s_hi) {
      float m = -INFINITY;
#pragma unroll
      for (int o = 0; o < 10; ++o) {
        z[o] += sb3[o];
        m = fmaxf(m, z[o]);
      }
      float se = 0.f;
#pragma unroll
      for (int o = 0; o < 10; ++o) se += expf(z[o] - m);
      const int lab = y[smp];
      float zl = z[0];
#pragma unroll
      for (int o = 1; o < 10; ++o) zl = o == lab ? z[o] : zl;
      loss = (m + logf(se)) - zl;
    }
    loss = warp_sum(loss);
    if (lane == 0) red[q] = loss;
  }
  tc_fence_before();
  __syncthreads();
  return ((red[0] + red[1]) + red[2]) + red[3];
}

__device__ __forceinline__ uint32_t tmem_alloc512(uint32_t* slot) {
  using namespace tc;
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  return *slot;
}
__device__ __forceinline__ void tmem_free512(uint32_t tmem) {
  using namespace tc;
  tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// k_lenet_fc_tc shared memory: f1w of the current candidate stays resident
// (one TMA load per candidate, i.e. per nparts items); the A operand streams
// through two buffers in K' parts of 144 / 144 / 128 (9 / 9 / 8 MMA k-steps).
__host__ __device__ constexpr int part_k(int p) { return p < 2 ? 144 : 128; }  // K' of part p
__host__ __device__ constexpr int part_k0(int p) { return 144 * p; }
constexpr int kA1PartBytes = 128 * 144 * 2;
struct FcTcSmem {
  static constexpr int w1 = 0;                           // f1w: 128 x 416 bf16
  static constexpr int a = w1 + kA1Bytes;                // 2 x A part: 128 x 144 bf16
  static constexpr int tail = a + 2 * kA1PartBytes;      // FcTail
  static constexpr int bar = tail + FcTail::bytes;       // u64: mma, w1, full[2], empty[2]
  static constexpr int slot = bar + 48;                  // TMEM base
  static constexpr int total = slot + 8;
};
static_assert(FcTcSmem::total <= 227 * 1024 && FcTcSmem::a % 1024 == 0 && FcTcSmem::tail % 16 == 0 &&
                  FcTcSmem::bar % 8 == 0,
              "LeNet fc shared memory");

}  // namespace

// k_lenet_fc_tc — split path: work item = (candidate, 128-sample chunk); the
// A operand = the chunk's pooled conv2 rows from the scratch, streamed by TMA
// (tmap_p2: 2-D view (K', sample row) of the scratch; a box (8, 128) is one
// K' chunk of 128 rows) in three K' parts through two buffers, so the loads
// of part n + 1 / n + 2 overlap the MMAs of part n and the fc tail of the
// item; f1w (tmap_f1) is loaded once per candidate and stays resident.
// Thread 0 is the TMA producer and the MMA issuer; all 8 warps run the
// epilogues.
__global__ void __launch_bounds__(kFcThreadsTc, 1) k_lenet_fc_tc(LenetSplitArgs sa,
                                                                 const __grid_constant__ CUtensorMap tmap_p2,
                                                                 const __grid_constant__ CUtensorMap tmap_f1) {
  using namespace tc;
  pdl_enter();
  const LenetArgs& args = sa.base;
  if (args.gate != nullptr && *args.gate == 0) return;
  extern __shared__ __align__(1024) uint8_t smem_fc[];
  uint8_t* tail = smem_fc + FcTcSmem::tail;
  const uint32_t bar_m = smem_u32(smem_fc + FcTcSmem::bar), bar_w = bar_m + 8, bar_full = bar_m + 16,
                 bar_empty = bar_m + 32;
  if (threadIdx.x == 0) {
    mbar_init(bar_m, 1);
    mbar_init(bar_w, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_full + 8 * b, 1);
      mbar_init(bar_empty + 8 * b, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_p2)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_f1)));
  }
  const uint32_t tmem = tmem_alloc512(reinterpret_cast<uint32_t*>(smem_fc + FcTcSmem::slot));
  const uint32_t w1_s = smem_u32(smem_fc + FcTcSmem::w1), a_s = smem_u32(smem_fc + FcTcSmem::a);
  MmaBar mb{bar_m, 0};

  const uint64_t total = args.rows * args.nparts;
  const uint64_t t_begin = total * blockIdx.x / gridDim.x;
  const uint64_t t_end = total * (blockIdx.x + 1) / gridDim.x;
  const uint64_t nseq = (t_end - t_begin) * 3;  // (item, K' part) sequence of this CTA
  // TMA of sequence entry n into buffer n % 2 (thread 0)
  auto load_part = [&](uint64_t n) {
    const uint64_t it = t_begin + n / 3;
    const int p = (int)(n % 3);
    const int srow = (int)((it / args.nparts) * args.S + (it % args.nparts) * kChunkS);
    const uint32_t dst = a_s + (uint32_t)(n & 1) * kA1PartBytes, fb = bar_full + 8 * (uint32_t)(n & 1);
    mbar_expect_tx(fb, (uint32_t)part_k(p) * 256);
    for (int cc = 0; cc < part_k(p) / 8; ++cc) tma_load_2d(dst + cc * 2048, &tmap_p2, fb, part_k0(p) + 8 * cc, srow);
  };
  if (threadIdx.x == 0) {
    if (nseq > 0) load_part(0);
    if (nseq > 1) load_part(1);
  }
  uint32_t pw = 0, pfull[2] = {0, 0}, pempty[2] = {0, 0};
  uint64_t staged = ~0ull;
  for (uint64_t item = t_begin; item < t_end; ++item) {
    const uint64_t row = item / args.nparts;
    const uint32_t part = (uint32_t)(item % args.nparts);
    const uint32_t s_lo = part * kChunkS, s_hi = min(args.S, s_lo + kChunkS);
    if (row != staged) {  // every MMA reading f1w / f2w / f3w of the previous candidate is complete
      if (threadIdx.x == 0) {
        mbar_expect_tx(bar_w, (uint32_t)kA1Bytes);
        for (int cc = 0; cc < kF1K / 8; ++cc)
          tma_load_3d(w1_s + cc * 2048, &tmap_f1, bar_w, 8 * cc, 0, (int)(sa.row0 + row));
      }
      stage_fc_tail(tail, args.W + row * args.Dp, kFcThreadsTc);
      __syncthreads();
      if (threadIdx.x == 0) {
        mbar_wait(bar_w, pw);
        pw ^= 1;
      }
      staged = row;
    }
    if (threadIdx.x == 0) {
      const uint64_t n0 = (item - t_begin) * 3;
      for (int p = 0; p < 3; ++p) {
        const uint64_t n = n0 + p;
        const uint32_t b = (uint32_t)(n & 1);
        mbar_wait(bar_full + 8 * b, pfull[b]);
        pfull[b] ^= 1;
        tc_fence_after();
        constexpr uint32_t id1 = idesc_bf16(128, 128);
        const int kk0 = part_k0(p) / 16;
        for (int kk = 0; kk < part_k(p) / 16; ++kk)
          mma_ss(tmem + kColD1, interleaved_desc(a_s + b * kA1PartBytes + kk * 2 * 2048, 2048, 128),
                 interleaved_desc(w1_s + (kk0 + kk) * 2 * 2048, 2048, 128), id1, (kk0 + kk) != 0);
        mma_commit(bar_empty + 8 * b);
        if (p == 2) mma_commit(bar_m);  // fc1 of the item complete
        if (n + 2 < nseq) {             // refill this buffer once its MMAs are done
          mbar_wait(bar_empty + 8 * b, pempty[b]);
          pempty[b] ^= 1;
          load_part(n + 2);
        } else {
          mbar_wait(bar_empty + 8 * b, pempty[b]);
          pempty[b] ^= 1;
        }
      }
    }
    mb.wait();  // fc1 done
    const float loss = fc_tail(tmem, tail, mb, s_lo, s_hi, args.y);
    if (threadIdx.x == 0) {
      args.part[(row * args.nparts + part) * 2] = loss;
      args.part[(row * args.nparts + part) * 2 + 1] = 0.0f;
    }
  }
  tmem_free512(tmem);
}

// ============================================================ fused kernel
// k_lenet_fused (MGFWA_LENET_FUSED=1) — the conv and the fc stack in one CTA
// per SM with no activation scratch in HBM: 8 conv warps write each
// sample's pooled conv2 output straight into the fc1 A operand in shared
// memory, then the item's fc stack runs as in k_lenet_fc_tc with the f1w
// halves staged through the conv buffers.  Measured slower than the split
// path (C3 fitness 6.77 vs 6.40 ms → see DESIGN.md): 8 conv warps instead of
// 12 (shared memory) cost more than the scratch round trip.
namespace {

#ifndef LENET_PROBE
#define LENET_PROBE 0  // 1: profiling probe, conv only (fc stage skipped, partials 0)
#endif
constexpr int kFW = 8;
constexpr int kFThreads = kFW * 32;
static_assert(kFThreads == kFcThreadsTc, "fc_tail expects 256 threads");

struct FusedSmem {
  static constexpr int wc1 = 0;                                  // [8][32] bf16
  static constexpr int wc2 = wc1 + 8 * kC1K * 2;                 // [16][216] bf16
  static constexpr int bc1 = wc2 + 16 * kC2S * 2;                // f32 [8]
  static constexpr int bc2 = bc1 + 8 * 4;                        // f32 [16]
  static constexpr int img = (bc2 + 16 * 4 + 127) / 128 * 128;   // per warp [33][40] u32 | f1w half (TMA dst)
  static constexpr int p1 = img + kFW * kImgWords * 4;           // per warp [14][kP1R][4] u32
  static constexpr int a1 = p1 + kFW * kP1Words * 4;             // fc1 A: 128 x 416 bf16
  static constexpr int tail = a1 + kA1Bytes;                     // FcTail
  static constexpr int bar = tail + FcTail::bytes;               // u64: MMA commit, TMA
  static constexpr int slot = bar + 16;                          // TMEM base
  static constexpr int total = slot + 8;
};
static_assert(FusedSmem::total <= 227 * 1024 && FusedSmem::a1 % 16 == 0 && FusedSmem::tail % 16 == 0 &&
                  FusedSmem::bar % 8 == 0,
              "fused LeNet shared memory");
static_assert(kW1HalfBytes <= FusedSmem::a1 - FusedSmem::img, "an f1w half fits the conv buffers");

}  // namespace

__global__ void __launch_bounds__(kFThreads, 1) k_lenet_fused(LenetArgs args,
                                                              const __grid_constant__ CUtensorMap tmap_f1) {
  using namespace tc;
  pdl_enter();
  if (args.gate != nullptr && *args.gate == 0) return;
  extern __shared__ __align__(1024) uint8_t smem_fused[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int wi = g >> 1, dx = g & 1;
  __nv_bfloat16* wc1 = reinterpret_cast<__nv_bfloat16*>(smem_fused + FusedSmem::wc1);
  __nv_bfloat16* wc2 = reinterpret_cast<__nv_bfloat16*>(smem_fused + FusedSmem::wc2);
  float* bc1 = reinterpret_cast<float*>(smem_fused + FusedSmem::bc1);
  float* bc2 = reinterpret_cast<float*>(smem_fused + FusedSmem::bc2);
  const uint32_t* img = reinterpret_cast<const uint32_t*>(smem_fused + FusedSmem::img) + warp * kImgWords;
  const uint32_t img_s = smem_addr(img);
  uint32_t* p1 = reinterpret_cast<uint32_t*>(smem_fused + FusedSmem::p1) + warp * kP1Words;
  __nv_bfloat16* a1 = reinterpret_cast<__nv_bfloat16*>(smem_fused + FusedSmem::a1);
  uint8_t* tail = smem_fused + FusedSmem::tail;
  const uint32_t bar = smem_u32(smem_fused + FusedSmem::bar), bar_tma = bar + 8;
  {
    uint32_t* p = reinterpret_cast<uint32_t*>(smem_fused);
    for (int i = threadIdx.x; i < FusedSmem::bar / 4; i += kFThreads) p[i] = 0u;
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar_tma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_f1)));
  }
  const uint32_t tmem = tmem_alloc512(reinterpret_cast<uint32_t*>(smem_fused + FusedSmem::slot));
  const uint32_t r_s = smem_u32(smem_fused + FusedSmem::img), a1_s = smem_u32(a1);
  MmaBar mb{bar, 0};
  uint32_t tphase = 0;

  const uint32_t* imgc = img + c * kImgS;
  const uint32_t* imgd = img + 4 * kImgS + 2 * (c < 3 ? c : 2);
  const uint32_t* p1c = p1 + c;
  const uint64_t total = args.rows * args.nparts;
  const uint64_t t_begin = total * blockIdx.x / gridDim.x;
  const uint64_t t_end = total * (blockIdx.x + 1) / gridDim.x;
  uint64_t staged = ~0ull;
  uint32_t bw1[2][2], bw2[13][2][2];
  float b1a = 0.f, b1b = 0.f, b2a = 0.f, b2b = 0.f, b2c = 0.f, b2d = 0.f;
  for (uint64_t item = t_begin; item < t_end; ++item) {
    const uint64_t row = item / args.nparts;
    const uint32_t part = (uint32_t)(item % args.nparts);
    const uint32_t s_lo = part * kChunkS, s_hi = min(args.S, s_lo + kChunkS);
    const __nv_bfloat16* w = args.W + row * args.Dp;
    __syncthreads();  // the previous item's readers of every buffer are done
    if (row != staged) {
      // conv weights / biases pre-scaled by 1/4 (average pools = sums of ReLUs)
      for (int i = threadIdx.x; i < 150; i += kFThreads) {
        const int ch = i / 25, r = i % 25, ky = r / 5, kx = r % 5;
        wc1[ch * kC1K + conv1_k(ky, kx)] = __float2bfloat16(0.25f * bf(w[oC1W + i]));
      }
      for (int i = threadIdx.x; i < 2400; i += kFThreads) {
        const int ch = i / 150, r = i % 150, ci = r / 25, tap = r % 25;
        wc2[ch * kC2S + conv2_k(tap / 5, tap % 5) + ci] = __float2bfloat16(0.25f * bf(w[oC2W + i]));
      }
      if (threadIdx.x < 6) bc1[threadIdx.x] = 0.25f * bf(w[oC1B + threadIdx.x]);
      if (threadIdx.x < 16) bc2[threadIdx.x] = 0.25f * bf(w[oC2B + threadIdx.x]);
      stage_fc_tail(tail, w, kFThreads);
      __syncthreads();
      staged = row;
#pragma unroll
      for (int st = 0; st < 2; ++st) {
        const __nv_bfloat16* b = wc1 + g * kC1K + 16 * st + 2 * c;
        bw1[st][0] = *reinterpret_cast<const uint32_t*>(b);
        bw1[st][1] = *reinterpret_cast<const uint32_t*>(b + 8);
      }
#pragma unroll
      for (int st = 0; st < 13; ++st)
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          const __nv_bfloat16* b = wc2 + (8 * n + g) * kC2S + 16 * st + 2 * c;
          bw2[st][n][0] = *reinterpret_cast<const uint32_t*>(b);
          bw2[st][n][1] = *reinterpret_cast<const uint32_t*>(b + 8);
        }
      b1a = bc1[2 * c], b1b = bc1[2 * c + 1];
      b2a = bc2[2 * c], b2b = bc2[2 * c + 1], b2c = bc2[8 + 2 * c], b2d = bc2[9 + 2 * c];
    }
    // ---- conv for the chunk's samples -> fc1 A operand
    if (s_lo + warp < s_hi) prefetch_img(img_s, args.pimg + (uint64_t)(s_lo + warp) * kImgWords, lane);
    for (uint32_t s = s_lo + warp; s < s_hi; s += kFW) {
      cp_async_wait_all();
      __syncwarp();
#pragma unroll 1
      for (int t0 = 0; t0 + LENET_CV_P1T <= 25; t0 += LENET_CV_P1T)
        conv1_pairs<LENET_CV_P1T>(t0, imgc, imgd, p1, g, c, bw1, b1a, b1b);
      if constexpr (25 % LENET_CV_P1T != 0)
        conv1_pairs<25 % LENET_CV_P1T>(25 - 25 % LENET_CV_P1T, imgc, imgd, p1, g, c, bw1, b1a, b1b);
      __syncwarp();
      if (s + kFW < s_hi) prefetch_img(img_s, args.pimg + (uint64_t)(s + kFW) * kImgWords, lane);
      const uint32_t r = s - s_lo;
      __nv_bfloat16* orow = a1 + ((r >> 3) * 128 + (r & 7) * 16) / 2;
#pragma unroll 1
      for (int t0 = 0; t0 + kCvC2T <= 7; t0 += kCvC2T)
        conv2_tiles<kCvC2T, true>(t0, p1c, orow, wi, dx, c, bw2, b2a, b2b, b2c, b2d);
      if constexpr (7 % kCvC2T != 0)
        conv2_tiles<7 % kCvC2T, true>(7 - 7 % kCvC2T, p1c, orow, wi, dx, c, bw2, b2a, b2b, b2c, b2d);
      __syncwarp();
    }
    async_smem_fence();  // generic-proxy writes of the A operand -> visible to the tensor core
    __syncthreads();
#if LENET_PROBE == 1
    if (threadIdx.x == 0) {
      args.part[(row * args.nparts + part) * 2] = 0.0f;
      args.part[(row * args.nparts + part) * 2 + 1] = 0.0f;
    }
    continue;
#endif
    // ---- fc1 with f1w in two TMA halves through the conv buffers, then the fc tail
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      if (threadIdx.x == 0) {
        mbar_expect_tx(bar_tma, (uint32_t)kW1HalfBytes);
        for (int cc = 0; cc < kF1Half / 8; ++cc)
          tma_load_3d(r_s + cc * 2048, &tmap_f1, bar_tma, h * kF1Half + 8 * cc, 0, (int)row);
      }
      mbar_wait(bar_tma, tphase);
      tphase ^= 1;
      if (threadIdx.x == 0) fc1_mma(tmem, a1_s, r_s, 13 * h, 13 * h + 13, 13 * h, bar);
      mb.wait();  // also frees the f1w half buffer
    }
    const float loss = fc_tail(tmem, tail, mb, s_lo, s_hi, args.y);
    if (threadIdx.x == 0) {
      args.part[(row * args.nparts + part) * 2] = loss;
      args.part[(row * args.nparts + part) * 2 + 1] = 0.0f;
    }
  }
  tmem_free512(tmem);
}

// ============================================================ conv1 on tcgen05
// k_lenet_conv_tc (default conv stage of the split path) — conv1 of a group
// of kCtG = 12 candidates as ONE tcgen05 GEMM per sample, conv2 per
// candidate on the warp MMA, pooled conv2 rows -> the scratch (same K' rows
// as k_lenet_conv, so k_lenet_fc_tc is unchanged).
//
// conv1 is transposed so that the shared operand is the image:
//   D[(candidate, channel), pixel] = A[(candidate, channel), k] . B[pixel, k]
//   M = 128 rows (72 used: row 32 q + j, q = 1..3, j < 24, is (candidate,
//       channel) = divmod(24 (q - 1) + j, 6); lane quarter 0 is empty, so
//       three epilogue warps cover the live rows),
//   K = 48 = 6 chunks of 8: chunk ky holds taps kx = 0..4, two zero taps and
//       a constant-1 tap (k = 7) that carries the bias in chunk 0,
//   N = 64 per MMA block = the two output pixel rows of one pooled row, 32
//       pixel slots each (28 used).
// The B operand is a "row-window" image precomputed once per plan:
// R[s][Y][X] = 16 bytes = (p[Y][X .. X+4], 0, 0, 1) with p the zero-padded
// 32 x 32 image.  In the no-swizzle K-major layout (8-row x 16-byte core
// matrices) the 8 pixels x0 .. x0+7 of one row are 128 contiguous bytes, the
// next 8 pixels follow (SBO = 128), and the next tap row ky + 1 is the next
// image row (LBO = 512 bytes): an implicit im2col with no replication beyond
// the 8-tap window, 16.9 KB per sample, one bulk copy.
// D blocks (128 lanes x 64 columns) cycle through 8 TMEM slots; a thread of
// the epilogue owns one (candidate, channel) row, so the 2 x 2 average pool
// (weights and bias pre-scaled by 1/4: a sum of four ReLUs) is in registers:
// column dy * 32 + x of the block.  Pooled rows land in the candidate's conv1
// map in shared memory (3-word pixels, see conv2_cols_tiles; kCtP = 4
// buffers), and conv2_cols_tiles consumes them: one warp per candidate with
// its conv2 B fragments in registers, loaded straight from the candidate row.
// The conv2 warps take the samples in pairs so that the two partial 7th tiles
// (pool window 24 alone) share one MMA tile: 13 instead of 14 tiles per two
// samples; each D row depends only on its own A row, so the fitness does not
// depend on the pairing.
//
// Warps (16, i.e. 4 per SM sub-partition, 128 registers): 0 = control
// (row-window bulk copies, conv1 A staging per group, lane 0 issues the
// MMAs), 1..3 = TMEM epilogue (lane quarter = warp), 4..15 = conv2.  Work = the (group, sample) units of the launch, split into equal
// contiguous ranges per CTA (group changes restage A and the fragments).
namespace {

constexpr int kCtG = 12;                               // candidates per conv1 GEMM
constexpr int kQR = 48;                                // conv1 map row stride (words), see conv2_cols_tiles
constexpr int kQCand = 14 * kQR + 8;                   // candidate stride (words; 8 mod 32: conflict-free epilogue stores)
#ifndef LENET_CT_C2T
#define LENET_CT_C2T 2
#endif
constexpr int kCtC2T = LENET_CT_C2T;                   // conv2 tiles in flight per warp
constexpr int kRwRows = 33, kRwPitch = 32;             // row windows: [Y][X] x 16 B
constexpr int kRwBytes = kRwRows * kRwPitch * 16;      // 16,896 B per sample
constexpr int kCtA = 128 * 48 * 2;                     // conv1 A: 128 x 48 bf16
constexpr int kCtSlots = 8;                            // TMEM: 8 x 64 columns
#ifndef LENET_CT_MAPS
#define LENET_CT_MAPS 4  // conv1-map buffers (a power of two: buffer / phase by mask and shift)
#endif
#ifndef LENET_CT_PAIR
#define LENET_CT_PAIR 1  // conv2 takes samples in pairs (shared 7th tile); needs LENET_CT_MAPS >= 3
#endif
static_assert(!LENET_CT_PAIR || LENET_CT_MAPS >= 3, "pairs need a third conv1-map buffer");
constexpr int kCtP = LENET_CT_MAPS;                    // conv1-map buffers (samples in flight)
constexpr int kCtWarps = 1 + 3 + kCtG;
constexpr int kCtThreads = kCtWarps * 32;
struct CtSmem {
  static constexpr int a = 0;                                   // 2 x conv1 A (group parity)
  static constexpr int rw = a + 2 * kCtA;                       // 2 x row windows (sample parity)
  static constexpr int p1 = rw + 2 * kRwBytes;                  // kCtP x kCtG conv1 maps (kQCand words each)
  static constexpr int o = p1 + kCtP * kCtG * kQCand * 4;       // per conv2 warp: 2 x [416] bf16
  static constexpr int bar = o + kCtG * 2 * kP2Row * 2;         // mbarriers
  // a_full[2] a_empty[2] rw_full[2] rw_empty[2] t_full[8] t_empty[8] p_full[kCtP] p_empty[kCtP]
  static constexpr int nbar = 24 + 2 * kCtP;
  static constexpr int slot = bar + nbar * 8;
  static constexpr int total = slot + 16;
};
static_assert(CtSmem::total <= 227 * 1024 && CtSmem::rw % 16 == 0 && CtSmem::o % 16 == 0 &&
                  CtSmem::bar % 8 == 0,
              "LeNet tcgen05 conv shared memory");
enum { kBaFull = 0, kBaEmpty = 2, kBrFull = 4, kBrEmpty = 6, kBtFull = 8, kBtEmpty = 16, kBpFull = 24, kBpEmpty = 24 + kCtP };

// (candidate, channel) of conv1 GEMM row r, or -1 for a padding row
__host__ __device__ constexpr int ct_row_cc(int r) {
  return (r >> 5) > 0 && (r & 31) < 24 ? 24 * ((r >> 5) - 1) + (r & 31) : -1;
}

struct LenetCtArgs {
  LenetSplitArgs sa;
  const uint8_t* rwin;  // [S][kRwBytes] row-window images
  uint64_t ngroups;     // ceil(rows / kCtG)
};

// conv2 of k_lenet_conv_tc in "column" K order.  The conv1 map of a
// candidate is [14 rows][16 pixel slots][3 channel pairs] words (kQR = 48
// words per row, slots 14 / 15 zero), so tap column col = kx * 3 + cp (the
// channel pair) is word offset col from the pixel and tap row ky is ky * kQR.
// K = 10 k-steps of 8 (column, ky) pairs:
//   steps 0-3 (A s) and 4-7 (B s): slots j < 4 = (col 4 s + j, ky0),
//     j >= 4 = (col 4 s + j - 4, ky0 + 1), ky0 = 0 (A) / 2 (B);
//   steps 8-9 (C h): slots j = (col 8 h + j, ky 4);
// column 15 is padding (zero weights, reads the zero slot 14 of the row).
// Lane c of an A / B step then needs, for its column, the words at ky0,
// ky0 + 1 (twice: row g + 8 at ky0 is row g at ky0 + 1, the pixel one row
// down) and ky0 + 2, and its C step the words at ky 4 / 5 of two columns: 24
// shared-memory loads per 16-pixel tile feed 20 MMAs (conv2_tiles: 30 loads,
// 26 MMAs).  With 3-word pixels and the 48-word row stride the 32 lanes of
// every load hit distinct banks (checked exhaustively over the 7 tiles).

__device__ __forceinline__ void conv2_slot(int step, int j, int& col, int& ky) {
  if (step < 4) {
    col = 4 * step + (j & 3), ky = j >> 2;
  } else if (step < 8) {
    col = 4 * (step - 4) + (j & 3), ky = 2 + (j >> 2);
  } else {
    col = 8 * (step - 8) + j, ky = 4;
  }
}

// B fragments of candidate row w in that K order, read straight from the row
// (weights and biases pre-scaled by 1/4, exact)
__device__ __forceinline__ void load_conv2_cols(const __nv_bfloat16* w, int g, int c, uint32_t (&bw)[10][2][2],
                                                float& b2a, float& b2b, float& b2c, float& b2d) {
  auto wv = [&](int ch, int col, int ky, int half) -> float {
    if (col >= 15) return 0.f;
    const int kx = col / 3, ci = 2 * (col % 3) + half;
    return 0.25f * bf(w[oC2W + ch * 150 + ci * 25 + ky * 5 + kx]);
  };
#pragma unroll
  for (int st = 0; st < 10; ++st)
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      const int ch = 8 * n + g;
      int col, ky;
      conv2_slot(st, c, col, ky);
      bw[st][n][0] = pack_bf16(wv(ch, col, ky, 0), wv(ch, col, ky, 1));
      conv2_slot(st, c + 4, col, ky);
      bw[st][n][1] = pack_bf16(wv(ch, col, ky, 0), wv(ch, col, ky, 1));
    }
  b2a = 0.25f * bf(w[oC2B + 2 * c]), b2b = 0.25f * bf(w[oC2B + 2 * c + 1]);
  b2c = 0.25f * bf(w[oC2B + 8 + 2 * c]), b2d = 0.25f * bf(w[oC2B + 9 + 2 * c]);
}

// conv2 + ReLU + pool of tiles t0 .. t0 + N - 1 (the conv2_tiles M layout:
// rows g / g + 8 = vertically adjacent pixels of window 4 t + g / 2) -> o
// PAIR (N = 1): the partial 7th tiles of two samples of the same candidate
// as one tile — window slot wi = 0 / 1 is pool window 24 of sample `map` /
// `map2` (outputs to o / o2), slots 2 / 3 repeat them (discarded).
template <int N, bool PAIR = false>
__device__ __forceinline__ void conv2_cols_tiles(int t0, const uint32_t* map, __nv_bfloat16* o, int wi, int dx,
                                                 int c, const uint32_t (&bw)[10][2][2], float b2a, float b2b,
                                                 float b2c, float b2d, const uint32_t* map2 = nullptr,
                                                 __nv_bfloat16* o2 = nullptr) {
  static_assert(!PAIR || N == 1, "one paired tile");
  int wv[N];
  const uint32_t* q[N];
  float d[N][2][4];
#pragma unroll
  for (int u = 0; u < N; ++u) {
    const int w = PAIR ? 24 : 4 * (t0 + u) + wi;
    wv[u] = PAIR ? (wi < 2 ? 24 : -1) : (w < 25 ? w : -1);
    const int wc = w < 25 ? w : 24;
    const int qy = wc / 5, qx = wc - 5 * qy;
    q[u] = (PAIR && (wi & 1) ? map2 : map) + (2 * qy) * kQR + (2 * qx + dx) * 3 + c;
    d[u][0][0] = b2a, d[u][0][1] = b2b, d[u][0][2] = b2a, d[u][0][3] = b2b;
    d[u][1][0] = b2c, d[u][1][1] = b2d, d[u][1][2] = b2c, d[u][1][3] = b2d;
  }
#pragma unroll
  for (int sp = 0; sp < 2; ++sp) {
    uint32_t W[N][2][6];
#pragma unroll
    for (int u = 0; u < N; ++u)
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int ky = 0; ky < 6; ++ky) W[u][e][ky] = q[u][ky * kQR + 4 * (2 * sp + e)];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int st = 2 * sp + e;
#pragma unroll
      for (int u = 0; u < N; ++u)
#pragma unroll
        for (int n = 0; n < 2; ++n)
          mma_bf16(d[u][n], W[u][e][0], W[u][e][1], W[u][e][1], W[u][e][2], bw[st][n][0], bw[st][n][1]);
#pragma unroll
      for (int u = 0; u < N; ++u)
#pragma unroll
        for (int n = 0; n < 2; ++n)
          mma_bf16(d[u][n], W[u][e][2], W[u][e][3], W[u][e][3], W[u][e][4], bw[4 + st][n][0], bw[4 + st][n][1]);
    }
#pragma unroll
    for (int u = 0; u < N; ++u)
#pragma unroll
      for (int n = 0; n < 2; ++n)
        mma_bf16(d[u][n], W[u][0][4], W[u][0][5], W[u][1][4], W[u][1][5], bw[8 + sp][n][0], bw[8 + sp][n][1]);
  }
#pragma unroll
  for (int u = 0; u < N; ++u) {
    float s0 = fmaxf(d[u][0][0], 0.f) + fmaxf(d[u][0][2], 0.f);
    float s1 = fmaxf(d[u][0][1], 0.f) + fmaxf(d[u][0][3], 0.f);
    float s2 = fmaxf(d[u][1][0], 0.f) + fmaxf(d[u][1][2], 0.f);
    float s3 = fmaxf(d[u][1][1], 0.f) + fmaxf(d[u][1][3], 0.f);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 4);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 4);
    s2 += __shfl_xor_sync(0xffffffffu, s2, 4);
    s3 += __shfl_xor_sync(0xffffffffu, s3, 4);
    if (dx == 0 && wv[u] >= 0) {
      const int w = wv[u];
      const float vals[4] = {s0, s1, s2, s3};
      const int chs[4] = {2 * c, 2 * c + 1, 8 + 2 * c, 9 + 2 * c};
      __nv_bfloat16* ou = PAIR && (wi & 1) ? o2 : o;
#pragma unroll
      for (int j = 0; j < 4; ++j) ou[chs[j] * 25 + w + 4] = __float2bfloat16(vals[j]);
    }
  }
}

}  // namespace

// Row-window images of the dataset (see k_lenet_conv_tc): R[s][Y][X] =
// (p[Y][X + e], e < 5; 0; 0; 1) with p[Y][X] = x[s][Y - 2][X - 2] (0 outside).
__global__ void k_lenet_rowwin(const __nv_bfloat16* X, uint32_t S, uint4* R) {
  const uint64_t n = (uint64_t)S * kRwRows * kRwPitch;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = i / (kRwRows * kRwPitch);
    const int r = (int)(i % (kRwRows * kRwPitch)), Y = r / kRwPitch, Xc = r % kRwPitch;
    const __nv_bfloat16* img = X + s * 784;
    uint16_t v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int yy = Y - 2, xx = Xc + e - 2;
      __nv_bfloat16 t = __float2bfloat16(e == 7 ? 1.0f : 0.0f);
      if (e < 5 && yy >= 0 && yy < 28 && xx >= 0 && xx < 28) t = img[yy * 28 + xx];
      v[e] = *reinterpret_cast<uint16_t*>(&t);
    }
    R[i] = make_uint4(v[0] | (uint32_t)v[1] << 16, v[2] | (uint32_t)v[3] << 16, v[4] | (uint32_t)v[5] << 16,
                      v[6] | (uint32_t)v[7] << 16);
  }
}

__global__ void __launch_bounds__(kCtThreads, 1) k_lenet_conv_tc(LenetCtArgs ca) {
  using namespace tc;
  pdl_enter();
  const LenetSplitArgs& sa = ca.sa;
  const LenetArgs& args = sa.base;
  if (args.gate != nullptr && *args.gate == 0) return;
  extern __shared__ __align__(1024) uint8_t smem_ct[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base_s = smem_u32(smem_ct);
  const uint32_t bars = base_s + CtSmem::bar;
  auto bar = [&](int i) -> uint32_t { return bars + 8u * (uint32_t)i; };
  {
    uint32_t* p = reinterpret_cast<uint32_t*>(smem_ct);
    for (int i = threadIdx.x; i < CtSmem::bar / 4; i += kCtThreads) p[i] = 0u;
    async_smem_fence();  // the zero padding of the A operands is read by the tensor core
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBaFull + i), 32);
      mbar_init(bar(kBaEmpty + i), 1);
      mbar_init(bar(kBrFull + i), 1);
      mbar_init(bar(kBrEmpty + i), 1);
    }
    for (int i = 0; i < kCtP; ++i) {
      mbar_init(bar(kBpFull + i), 3 * 32);
      mbar_init(bar(kBpEmpty + i), kCtG * 32);
    }
    for (int i = 0; i < kCtSlots; ++i) {
      mbar_init(bar(kBtFull + i), 1);
      mbar_init(bar(kBtEmpty + i), 3 * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t tmem = tmem_alloc512(reinterpret_cast<uint32_t*>(smem_ct + CtSmem::slot));

  const uint64_t S = args.S;
  const uint64_t U = ca.ngroups * S;
  const uint64_t u0 = U * blockIdx.x / gridDim.x, u1 = U * (blockIdx.x + 1) / gridDim.x;
  const uint64_t n = u1 - u0;

  if (warp == 0) {
    // ---------------------------------------------------------- control: loads + conv1 MMAs
    constexpr uint32_t id = idesc_bf16(128, 64);
    // unit u = (group, sample) = divmod(u, S), stepped incrementally (no 64-bit divisions per sample)
    auto load_rw = [&](uint64_t i, uint64_t smp) {  // lane 0: row windows of unit i (sample smp) -> buffer i & 1
      const uint32_t b = (uint32_t)(i & 1);
      mbar_wait(bar(kBrEmpty + b), (uint32_t)((i >> 1) & 1) ^ 1);
      mbar_expect_tx(bar(kBrFull + b), kRwBytes);
      bulk_load(base_s + CtSmem::rw + b * kRwBytes, ca.rwin + smp * kRwBytes, kRwBytes, bar(kBrFull + b));
    };
    uint64_t grp = u0 / S, smp = u0 % S;
    if (lane == 0 && n > 0) load_rw(0, smp);
    uint64_t cur = ~0ull, tb = 0;
    int k = -1;
    for (uint64_t i = 0; i < n; ++i, (++smp == S ? (smp = 0, ++grp) : 0)) {
      if (grp != cur) {  // stage the group's conv1 A operand (buffer k & 1)
        if (lane == 0 && k >= 0) mma_commit(bar(kBaEmpty + (k & 1)));
        cur = grp;
        ++k;
        mbar_wait(bar(kBaEmpty + (k & 1)), ((k >> 1) & 1) ^ 1);
        uint8_t* A = smem_ct + CtSmem::a + (k & 1) * kCtA;
        for (int e = lane; e < 128 * 6; e += 32) {
          const int r = e / 6, ky = e - 6 * (e / 6);
          const int cc = ct_row_cc(r);
          uint16_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          if (cc >= 0 && ky < 5) {
            const int cand = cc / 6, ch = cc - 6 * (cc / 6);
            const uint64_t row = grp * kCtG + (uint64_t)cand;
            if (row < args.rows) {
              const __nv_bfloat16* w = args.W + row * args.Dp;
#pragma unroll
              for (int kx = 0; kx < 5; ++kx) {
                __nv_bfloat16 t = __float2bfloat16(0.25f * bf(w[oC1W + ch * 25 + ky * 5 + kx]));
                v[kx] = *reinterpret_cast<uint16_t*>(&t);
              }
              if (ky == 0) {
                __nv_bfloat16 t = __float2bfloat16(0.25f * bf(w[oC1B + ch]));
                v[7] = *reinterpret_cast<uint16_t*>(&t);
              }
            }
          }
          *reinterpret_cast<uint4*>(A + il_off(r, 8 * ky, 128)) =
              make_uint4(v[0] | (uint32_t)v[1] << 16, v[2] | (uint32_t)v[3] << 16, v[4] | (uint32_t)v[5] << 16,
                         v[6] | (uint32_t)v[7] << 16);
        }
        async_smem_fence();
        __syncwarp();
      }
      if (lane == 0) {
        if (i + 1 < n) load_rw(i + 1, smp + 1 == S ? 0 : smp + 1);
        const uint32_t b = (uint32_t)(i & 1);
        mbar_wait(bar(kBrFull + b), (uint32_t)(i >> 1) & 1);
        tc_fence_after();
        const uint32_t a_s = base_s + CtSmem::a + (k & 1) * kCtA;
        const uint32_t r_s = base_s + CtSmem::rw + b * kRwBytes;
        for (int py = 0; py < 14; ++py, ++tb) {
          const uint32_t slot = (uint32_t)(tb % kCtSlots);
          mbar_wait(bar(kBtEmpty + slot), (uint32_t)((tb / kCtSlots) & 1) ^ 1);
          tc_fence_after();
#pragma unroll
          for (int j = 0; j < 3; ++j)
            mma_ss(tmem + slot * 64, interleaved_desc(a_s + j * 2 * 2048, 2048, 128),
                   interleaved_desc(r_s + (2 * py + 2 * j) * 512, 512, 128), id, j != 0);
          mma_commit(bar(kBtFull + slot));
        }
        mma_commit(bar(kBrEmpty + b));
      }
      __syncwarp();
    }
  } else if (warp < 4) {
    // ---------------------------------------------------------- TMEM epilogue: ReLU + pool -> conv1 maps
    const int q = warp & 3, r = 32 * q + lane;
    const int cc = ct_row_cc(r);
    const int cand = cc >= 0 ? cc / 6 : 0, ch = cc >= 0 ? cc - 6 * (cc / 6) : 0;
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
    uint64_t tb = 0;
    for (uint64_t i = 0; i < n; ++i) {
      const uint32_t b = (uint32_t)(i % kCtP);
      mbar_wait(bar(kBpEmpty + b), (uint32_t)((i / kCtP) & 1) ^ 1);
      uint16_t* p1h = reinterpret_cast<uint16_t*>(smem_ct + CtSmem::p1 + (b * kCtG + cand) * kQCand * 4) + (ch >> 1) * 2 +
                      (ch & 1);
      for (int py = 0; py < 14; ++py, ++tb) {
        const uint32_t slot = (uint32_t)(tb % kCtSlots);
        mbar_wait(bar(kBtFull + slot), (uint32_t)(tb / kCtSlots) & 1);
        tc_fence_after();
#pragma unroll
        for (int hx = 0; hx < 2; ++hx) {  // pixel columns [16 hx, 16 hx + 16) of both rows
          float v0[16], v2[16];
          tmem_ld16_nowait(tq + slot * 64 + 16 * hx, v0);
          tmem_ld16_nowait(tq + slot * 64 + 32 + 16 * hx, v2);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (hx == 1) {
            tc_fence_before();
            mbar_arrive(bar(kBtEmpty + slot));
          }
          if (cc >= 0) {
#pragma unroll
            for (int u = 0; u < (hx == 0 ? 8 : 6); ++u) {
              // window px = 8 hx + u: row dy = 0 in v0, dy = 1 in v2
              const float sum = (fmaxf(v0[2 * u], 0.f) + fmaxf(v2[2 * u], 0.f)) +
                                (fmaxf(v0[2 * u + 1], 0.f) + fmaxf(v2[2 * u + 1], 0.f));
              __nv_bfloat16 t = __float2bfloat16(sum);
              p1h[(py * kQR + (8 * hx + u) * 3) * 2] = *reinterpret_cast<uint16_t*>(&t);
            }
          }
        }
      }
      mbar_arrive(bar(kBpFull + b));
    }
  } else {
    // ---------------------------------------------------------- conv2 (one candidate per warp)
    const int w = warp - 4;
    const int g = lane >> 2, c = lane & 3;
    const int wi = g >> 1, dx = g & 1;
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(smem_ct + CtSmem::o) + w * 2 * kP2Row;
    const uint32_t* maps = reinterpret_cast<const uint32_t*>(smem_ct + CtSmem::p1) + w * kQCand;
    uint32_t bw[10][2][2];
    float b2a = 0.f, b2b = 0.f, b2c = 0.f, b2d = 0.f;
    uint64_t cur = ~0ull;
    // LENET_CT_PAIR: samples in pairs (same group) whose partial 7th tiles share one MMA tile
    uint64_t grp = u0 / S, s = u0 % S;  // unit i = (grp, s), stepped incrementally
    for (uint64_t i = 0; i < n;) {
      const bool pair = LENET_CT_PAIR && i + 1 < n && s + 1 < S;
      const uint64_t row = grp * kCtG + (uint64_t)w;
      const bool live = row < args.rows;
      if (grp != cur) {
        cur = grp;
        if (live) load_conv2_cols(args.W + row * args.Dp, g, c, bw, b2a, b2b, b2c, b2d);
      }
      const uint32_t b0 = (uint32_t)(i % kCtP), b1 = (uint32_t)((i + 1) % kCtP);
      mbar_wait(bar(kBpFull + b0), (uint32_t)(i / kCtP) & 1);
      if (pair) mbar_wait(bar(kBpFull + b1), (uint32_t)((i + 1) / kCtP) & 1);
      if (live) {
        const uint32_t* m0 = maps + b0 * kCtG * kQCand;
        const uint32_t* m1 = maps + b1 * kCtG * kQCand;
#pragma unroll 1
        for (int t0 = 0; t0 + kCtC2T <= 6; t0 += kCtC2T)
          conv2_cols_tiles<kCtC2T>(t0, m0, o, wi, dx, c, bw, b2a, b2b, b2c, b2d);
        if (pair) {
#pragma unroll 1
          for (int t0 = 0; t0 + kCtC2T <= 6; t0 += kCtC2T)
            conv2_cols_tiles<kCtC2T>(t0, m1, o + kP2Row, wi, dx, c, bw, b2a, b2b, b2c, b2d);
          conv2_cols_tiles<1, true>(6, m0, o, wi, dx, c, bw, b2a, b2b, b2c, b2d, m1, o + kP2Row);
        } else {
          conv2_cols_tiles<1>(6, m0, o, wi, dx, c, bw, b2a, b2b, b2c, b2d);
        }
      }
      mbar_arrive(bar(kBpEmpty + b0));
      if (pair) mbar_arrive(bar(kBpEmpty + b1));
      if (live) {
        __syncwarp();
        for (int k = 0; k < (pair ? 2 : 1); ++k) {
          uint4* dst = reinterpret_cast<uint4*>(sa.p2 + (row * S + s + k) * (uint64_t)kP2Row);
          const uint4* srcv = reinterpret_cast<const uint4*>(o + k * kP2Row);
          for (int e = lane; e < kP2Row * 2 / 16; e += 32) dst[e] = srcv[e];
        }
        __syncwarp();
      }
      const uint64_t adv = pair ? 2 : 1;
      i += adv;
      s += adv;
      if (s >= S) s -= S, ++grp;
    }
  }
  tmem_free512(tmem);
}

struct LenetPlan {
  LenetArgs args;
  bool fused;    // MGFWA_LENET_FUSED=1: k_lenet_fused; default: conv + k_lenet_fc_tc
  bool conv_tc;  // conv stage: k_lenet_conv_tc (default) or k_lenet_conv (MGFWA_LENET_CONV=mma)
  uint8_t* rwin; // owned: row-window images [S][kRwBytes]
  int nsm;
  unsigned grid;
  uint64_t group_rows;  // candidates per conv / fc launch pair (bounds the scratch)
  uint32_t* pimg;       // owned
  __nv_bfloat16* p2;    // owned scratch [group_rows][S][416]
  CUtensorMap tmap_f1, tmap_p2;
};

uint32_t lenet_num_parts(uint32_t S) { return (S + kChunkS - 1) / kChunkS; }
uint64_t lenet_dim() { return kLenetDim; }

LenetPlan* lenet_plan_create(const __nv_bfloat16* X, const int32_t* y, uint32_t S,
                             const __nv_bfloat16* W, uint64_t rows, uint64_t Dp, int nsm,
                             char* err, size_t errlen) {
  if (S == 0 || rows == 0) {
    snprintf(err, errlen, "LeNet objective: samples and rows must be positive");
    return nullptr;
  }
  if (Dp % 8 != 0 || Dp < (uint64_t)kLenetDim) {
    snprintf(err, errlen, "LeNet objective: bad row stride");
    return nullptr;
  }
  if (cudaFuncSetAttribute(k_lenet_conv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           ConvSmem::total) != cudaSuccess ||
      cudaFuncSetAttribute(k_lenet_fc_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           FcTcSmem::total) != cudaSuccess ||
      cudaFuncSetAttribute(k_lenet_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           FusedSmem::total) != cudaSuccess ||
      cudaFuncSetAttribute(k_lenet_conv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           CtSmem::total) != cudaSuccess) {
    snprintf(err, errlen, "LeNet objective: shared memory opt-in failed");
    return nullptr;
  }
  tc::EncodeTiledFn enc = tc::get_encode_fn();
  if (!enc) {
    snprintf(err, errlen, "LeNet objective: cuTensorMapEncodeTiled unavailable");
    return nullptr;
  }
  auto* p = new (std::nothrow) LenetPlan{};
  if (!p) return nullptr;
  auto fail = [&](const char* m) -> LenetPlan* {
    snprintf(err, errlen, "%s", m);
    lenet_plan_destroy(p);
    return nullptr;
  };
  if (cudaMalloc(&p->pimg, (size_t)S * kImgWords * 4) != cudaSuccess)
    return fail("LeNet objective: cudaMalloc of the pair images failed");
  const uint64_t n = (uint64_t)S * kImgWords;
  k_lenet_pairs<<<(unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256>>>(X, S, p->pimg);
  if (cudaDeviceSynchronize() != cudaSuccess) return fail("LeNet objective: pair-image kernel failed");
  p->args.pimg = p->pimg;
  p->args.y = y;
  p->args.W = W;
  p->args.rows = rows;
  p->args.Dp = Dp;
  p->args.S = S;
  p->args.nparts = lenet_num_parts(S);
  {
    cuuint64_t dims[3] = {404, 120, rows};
    cuuint64_t strides[2] = {800, Dp * 2};
    cuuint32_t box[3] = {8, 128, 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&p->tmap_f1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<__nv_bfloat16*>(W + oF1W - kF1Shift), dims,
            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail("LeNet objective: f1w tensor map encode failed");
  }
  {
    const char* e = getenv("MGFWA_LENET_FUSED");
    p->fused = e && e[0] == '1';
  }
  if (p->fused) {
    const uint64_t items = rows * p->args.nparts;
    p->grid = (unsigned)(items < (uint64_t)nsm ? items : (uint64_t)nsm);
    p->group_rows = rows;
    return p;
  }
  {
    // MGFWA_LENET_CONV=mma: the warp-MMA conv (k_lenet_conv) instead of
    // k_lenet_conv_tc.  One conv kernel per plan, so a candidate's fitness
    // does not depend on the size of the batch it is evaluated in.
    const char* e = getenv("MGFWA_LENET_CONV");
    p->conv_tc = !(e && strcmp(e, "mma") == 0);
  }
  p->nsm = nsm;
  if (p->conv_tc) {
    if (cudaMalloc(&p->rwin, (size_t)S * kRwBytes) != cudaSuccess)
      return fail("LeNet objective: cudaMalloc of the row-window images failed");
    const uint64_t m = (uint64_t)S * kRwRows * kRwPitch;
    k_lenet_rowwin<<<(unsigned)((m + 255) / 256 < 4096 ? (m + 255) / 256 : 4096), 256>>>(
        X, S, reinterpret_cast<uint4*>(p->rwin));
    if (cudaDeviceSynchronize() != cudaSuccess) return fail("LeNet objective: row-window kernel failed");
  }
  // scratch of at most kScratchBytes (at least one candidate's activations)
  const uint64_t per_row = (uint64_t)S * kP2Row * 2;
  uint64_t cap = kScratchBytes;
  if (const char* e = getenv("MGFWA_LENET_SCRATCH_MB"))  // tests: force candidate groups
    cap = (uint64_t)strtoull(e, nullptr, 10) << 20;
  p->group_rows = cap / per_row;
  if (p->group_rows < 1) p->group_rows = 1;
  if (p->group_rows > rows) p->group_rows = rows;
  if (cudaMalloc(&p->p2, p->group_rows * per_row) != cudaSuccess)
    return fail("LeNet objective: cudaMalloc of the activation scratch failed");
  {
    cuuint64_t dims[2] = {(cuuint64_t)kP2Row, p->group_rows * S};
    cuuint64_t strides[1] = {(cuuint64_t)kP2Row * 2};
    cuuint32_t box[2] = {8, 128};
    cuuint32_t es[2] = {1, 1};
    if (enc(&p->tmap_p2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p->p2, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail("LeNet objective: scratch tensor map encode failed");
  }
  const uint64_t items = p->group_rows * p->args.nparts;
  p->grid = (unsigned)(items < (uint64_t)nsm ? items : (uint64_t)nsm);
  return p;
}

void lenet_plan_destroy(LenetPlan* p) {
  if (!p) return;
  cudaFree(p->pimg);
  cudaFree(p->rwin);
  cudaFree(p->p2);
  delete p;
}

cudaError_t lenet_fitness_launch(const LenetPlan* p, float* part, const int* gate,
                                 cudaStream_t s) {
  if (p->fused) {
    LenetArgs a = p->args;
    a.part = part;
    a.gate = gate;
    return pdl_launch(k_lenet_fused, p->grid, kFThreads, FusedSmem::total, s, a, p->tmap_f1);
  }
  for (uint64_t r0 = 0; r0 < p->args.rows; r0 += p->group_rows) {
    LenetSplitArgs sa{p->args, r0, p->p2};
    sa.base.W += r0 * p->args.Dp;
    sa.base.rows = p->args.rows - r0 < p->group_rows ? p->args.rows - r0 : p->group_rows;
    sa.base.part = part + r0 * p->args.nparts * 2;
    sa.base.gate = gate;
    const uint64_t items = sa.base.rows * sa.base.nparts;
    const unsigned gc = (unsigned)(items < p->grid ? items : p->grid);
    cudaError_t e;
    if (p->conv_tc) {
      LenetCtArgs ca{sa, p->rwin, (sa.base.rows + kCtG - 1) / kCtG};
      const uint64_t units = ca.ngroups * sa.base.S;
      const unsigned gt = (unsigned)(units < (uint64_t)p->nsm ? units : (uint64_t)p->nsm);
      e = pdl_launch(k_lenet_conv_tc, gt, kCtThreads, CtSmem::total, s, ca);
    } else {
      e = pdl_launch(k_lenet_conv, gc, kConvThreads, ConvSmem::total, s, sa);
    }
    if (e != cudaSuccess) return e;
    e = pdl_launch(k_lenet_fc_tc, gc, kFcThreadsTc, FcTcSmem::total, s, sa, p->tmap_p2, p->tmap_f1);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace mgfwa_b200
