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
constexpr int kF1S = 408;   // fc1 row stride (bf16), 128 rows, K = 400 (window-major)
constexpr int kF2S = 136;   // fc2: 96 rows, K = 128 (120 + pad)
constexpr int kF3S = 104;   // fc3: 16 rows, K = 96 (84 + pad)
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
constexpr int kP2S = 408;   // pooled conv2 activations per sample (bf16), [25][16]
constexpr int kH1S = 136;
constexpr int kH2S = 104;

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

__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
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
constexpr int kP2Row = 400;  // bf16 per sample in the scratch
constexpr uint64_t kScratchBytes = 2ull << 30;  // activation scratch cap (C3: 1.23 GB)

struct ConvSmem {
  static constexpr int wc1 = 0;                                // [8][32] bf16
  static constexpr int wc2 = wc1 + 8 * kC1K * 2;               // [16][216] bf16
  static constexpr int bc1 = wc2 + 16 * kC2S * 2;              // f32 [8]
  static constexpr int bc2 = bc1 + 8 * 4;                      // f32 [16]
  static constexpr int img = bc2 + 16 * 4;                     // per warp [33][40] u32
  static constexpr int p1 = img + kConvWarps * kImgWords * 4;  // per warp [14][kP1R][4] u32
  static constexpr int p2 = p1 + kConvWarps * kP1Words * 4;    // per warp [400] bf16
  static constexpr int total = p2 + kConvWarps * kP2Row * 2;
};
static_assert(ConvSmem::img % 16 == 0 && ConvSmem::p2 % 16 == 0, "aligned cp.async / uint4 regions");

constexpr int kFcWarps = 8;
constexpr int kFcThreads = kFcWarps * 32;
struct FcSmem {
  static constexpr int r = 0;                            // [128][408] bf16: wf1 staging | p2 chunk
  static constexpr int wf2 = r + 128 * kF1S * 2;         // [96][136]
  static constexpr int wf3 = wf2 + 96 * kF2S * 2;        // [16][104]
  static constexpr int bf1 = wf3 + 16 * kF3S * 2;        // f32 [128]
  static constexpr int bf2 = bf1 + 128 * 4;              // f32 [96]
  static constexpr int bf3 = bf2 + 96 * 4;               // f32 [16]
  static constexpr int wsum = bf3 + 16 * 4;              // f32 [8]
  static constexpr int h1 = wsum + 8 * 4;                // [128][136] bf16 (then f32 logits [128][16])
  static constexpr int h2 = h1 + 128 * kH1S * 2;         // [128][104] bf16
  static constexpr int total = h2 + 128 * kH2S * 2;
};
static_assert(FcSmem::total <= 227 * 1024 && FcSmem::h1 % 16 == 0 && FcSmem::h2 % 16 == 0 &&
                  FcSmem::wf2 % 16 == 0 && FcSmem::wf3 % 16 == 0,
              "LeNet fc shared memory");
static_assert(kF1S == kP2S && kChunkS == 128, "the staging region doubles as the p2 chunk");

struct LenetSplitArgs {
  LenetArgs base;
  __nv_bfloat16* p2;  // [rows][S][400] scratch
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

// IL = false: o = the sample's [25 windows][16 channels] bf16 row (scratch
// path).  IL = true: o = the sample's row base inside the fc1 A operand of
// the fused kernel (tcgen05 no-swizzle K-major layout, K = ch * 25 + window,
// see fc1_a_off): each value goes straight to its slot.
template <int N, bool IL = false>
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
      if (IL) {
        // K = ch * 25 + w: byte (K / 8) * 2048 + (K % 8) * 2 from the row base
        const int w = wv[u];
        const float vals[4] = {s0, s1, s2, s3};
        const int chs[4] = {2 * c, 2 * c + 1, 8 + 2 * c, 9 + 2 * c};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = chs[q] * 25 + w;
          o[(k >> 3) * 1024 + (k & 7)] = __float2bfloat16(vals[q]);
        }
      } else {
        uint32_t* ow = reinterpret_cast<uint32_t*>(o + wv[u] * 16);
        ow[c] = pack_bf16(s0, s1);
        ow[4 + c] = pack_bf16(s2, s3);
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
      // ---- conv2 + ReLU + pool -> o (window-major [25][16]): 7 tiles
#pragma unroll 1
      for (int t0 = 0; t0 + kCvC2T <= 7; t0 += kCvC2T)
        conv2_tiles<kCvC2T>(t0, p1c, o, wi, dx, c, bw2, b2a, b2b, b2c, b2d);
      if constexpr (7 % kCvC2T != 0) conv2_tiles<7 % kCvC2T>(7 - 7 % kCvC2T, p1c, o, wi, dx, c, bw2, b2a, b2b, b2c, b2d);
      __syncwarp();
      // ---- p2 row -> scratch (800 B, coalesced 16-byte stores)
      uint4* dst = reinterpret_cast<uint4*>(sa.p2 + (row * args.S + s) * (uint64_t)kP2Row);
      const uint4* srcv = reinterpret_cast<const uint4*>(o);
      for (int i = lane; i < kP2Row * 2 / 16; i += 32) dst[i] = srcv[i];
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kFcThreads, 1) k_lenet_fc(LenetSplitArgs sa) {
  pdl_enter();
  const LenetArgs& args = sa.base;
  if (args.gate != nullptr && *args.gate == 0) return;
  extern __shared__ __align__(16) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  __nv_bfloat16* rg = reinterpret_cast<__nv_bfloat16*>(sm + FcSmem::r);  // wf1 staging | p2 chunk
  __nv_bfloat16* wf2 = reinterpret_cast<__nv_bfloat16*>(sm + FcSmem::wf2);
  __nv_bfloat16* wf3 = reinterpret_cast<__nv_bfloat16*>(sm + FcSmem::wf3);
  float* bf1 = reinterpret_cast<float*>(sm + FcSmem::bf1);
  float* bf2 = reinterpret_cast<float*>(sm + FcSmem::bf2);
  float* bf3 = reinterpret_cast<float*>(sm + FcSmem::bf3);
  __nv_bfloat16* h1 = reinterpret_cast<__nv_bfloat16*>(sm + FcSmem::h1);
  __nv_bfloat16* h2 = reinterpret_cast<__nv_bfloat16*>(sm + FcSmem::h2);
  float* logit = reinterpret_cast<float*>(sm + FcSmem::h1);  // [128][16], h1 is dead by then
  float* wsum = reinterpret_cast<float*>(sm + FcSmem::wsum);
  {
    uint32_t* p = reinterpret_cast<uint32_t*>(sm);
    for (int i = threadIdx.x; i < FcSmem::total / 4; i += kFcThreads) p[i] = 0u;
  }
  __syncthreads();
  // ldmatrix lane addressing: matrices {rows 0-7, k lo}, {rows 8-15, k lo},
  // {rows 0-7, k hi}, {rows 8-15, k hi} for A; {n 0-7, k lo}, {n 0-7, k hi},
  // {n 8-15, k lo}, {n 8-15, k hi} for two B n-tiles.
  const int a_row = (lane & 7) + ((lane >> 3) & 1) * 8, a_col = (lane >> 4) * 8;
  const int b_row = (lane & 7) + (lane >> 4) * 8, b_col = ((lane >> 3) & 1) * 8;
  const uint32_t r_s = smem_addr(rg), h1_s = smem_addr(h1), h2_s = smem_addr(h2);
  const uint32_t wf2_s = smem_addr(wf2), wf3_s = smem_addr(wf3);

  const uint64_t total = args.rows * args.nparts;
  const uint64_t t_begin = total * blockIdx.x / gridDim.x;
  const uint64_t t_end = total * (blockIdx.x + 1) / gridDim.x;
  uint64_t staged = ~0ull;
  uint32_t af1[25][4];  // this warp's fc1 A fragments (outputs 16 warp .. +15, K = 400)
  float bias1[2] = {0.f, 0.f};
  for (uint64_t item = t_begin; item < t_end; ++item) {
    const uint64_t row = item / args.nparts;
    const uint32_t part = (uint32_t)(item % args.nparts);
    const uint32_t s_lo = part * kChunkS, s_hi = min(args.S, s_lo + kChunkS);
    __syncthreads();  // previous item: readers of the region / h1 / logits are done
    if (row != staged) {
      const __nv_bfloat16* w = args.W + row * args.Dp;
      // window-major columns: task (j, win) gathers f1w[j][ch * 25 + win] for
      // the 16 channels (lanes read consecutive windows: coalesced) and
      // writes them as two 16-byte words
      for (int i = threadIdx.x; i < 120 * 25; i += kFcThreads) {
        const int j = i / 25, win = i - 25 * j;
        const __nv_bfloat16* src = w + oF1W + j * 400 + win;
        uint32_t u[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          __nv_bfloat162 t;
          t.x = src[(2 * q) * 25];
          t.y = src[(2 * q + 1) * 25];
          u[q] = *reinterpret_cast<uint32_t*>(&t);
        }
        uint4* dst = reinterpret_cast<uint4*>(rg + j * kF1S + win * 16);
        dst[0] = make_uint4(u[0], u[1], u[2], u[3]);
        dst[1] = make_uint4(u[4], u[5], u[6], u[7]);
      }
      for (int i = threadIdx.x; i < 8 * kF1S / 2; i += kFcThreads)  // rows 120..127 = 0
        reinterpret_cast<uint32_t*>(rg + 120 * kF1S)[i] = 0u;
      for (int i = threadIdx.x; i < 84 * 30; i += kFcThreads) {
        const int j = i / 30, q = i % 30;
        *reinterpret_cast<uint2*>(wf2 + j * kF2S + q * 4) =
            *reinterpret_cast<const uint2*>(w + oF2W + j * 120 + q * 4);
      }
      for (int i = threadIdx.x; i < 10 * 21; i += kFcThreads) {
        const int j = i / 21, q = i % 21;
        *reinterpret_cast<uint2*>(wf3 + j * kF3S + q * 4) =
            *reinterpret_cast<const uint2*>(w + oF3W + j * 84 + q * 4);
      }
      if (threadIdx.x < 120) bf1[threadIdx.x] = bf(w[oF1B + threadIdx.x]);
      if (threadIdx.x < 84) bf2[threadIdx.x] = bf(w[oF2B + threadIdx.x]);
      if (threadIdx.x < 10) bf3[threadIdx.x] = bf(w[oF3B + threadIdx.x]);
      __syncthreads();
      const uint32_t a_base = r_s + (uint32_t)(((16 * warp + a_row) * kF1S + a_col) * 2);
#pragma unroll
      for (int st = 0; st < 25; ++st) ldmatrix_x4(af1[st], a_base + st * 32);
      {
        const int j0 = 16 * warp + g, j1 = j0 + 8;
        bias1[0] = j0 < 120 ? bf1[j0] : 0.f;
        bias1[1] = j1 < 120 ? bf1[j1] : 0.f;
      }
      staged = row;
      __syncthreads();  // the region is about to hold activations
    }
    // ---- p2 rows of the chunk (cp.async, zero rows past s_hi)
    for (int i = threadIdx.x; i < (int)kChunkS * 50; i += kFcThreads) {
      const int r = i / 50, q = i % 50;
      const uint32_t dst = r_s + (uint32_t)(r * kP2S * 2 + q * 16);
      if (s_lo + r < s_hi)
        cp_async16(dst, sa.p2 + (row * args.S + s_lo + r) * (uint64_t)kP2Row + q * 8);
      else
        *reinterpret_cast<uint4*>(rg + r * kP2S + q * 8) = make_uint4(0u, 0u, 0u, 0u);
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    // ---- fc1: outputs 16 warp .. +15 for all 128 samples, 4 n-tiles at a time
#pragma unroll 1
    for (int ng = 0; ng < 16; ng += 4) {
      float d[4][4] = {};
      const uint32_t b_base = r_s + (uint32_t)(((8 * ng + b_row) * kP2S + b_col) * 2);
#pragma unroll
      for (int st = 0; st < 25; ++st) {
        uint32_t b[2][4];
        ldmatrix_x4(b[0], b_base + st * 32);
        ldmatrix_x4(b[1], b_base + 16 * kP2S * 2 + st * 32);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          mma_bf16(d[j], af1[st][0], af1[st][1], af1[st][2], af1[st][3], b[j >> 1][(j & 1) * 2],
                   b[j >> 1][(j & 1) * 2 + 1]);
      }
      const int j0 = 16 * warp + g, j1 = j0 + 8;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int s0 = 8 * (ng + j) + 2 * c;
        h1[s0 * kH1S + j0] = __float2bfloat16(j0 < 120 ? fmaxf(d[j][0] + bias1[0], 0.f) : 0.f);
        h1[(s0 + 1) * kH1S + j0] = __float2bfloat16(j0 < 120 ? fmaxf(d[j][1] + bias1[0], 0.f) : 0.f);
        h1[s0 * kH1S + j1] = __float2bfloat16(j1 < 120 ? fmaxf(d[j][2] + bias1[1], 0.f) : 0.f);
        h1[(s0 + 1) * kH1S + j1] = __float2bfloat16(j1 < 120 ? fmaxf(d[j][3] + bias1[1], 0.f) : 0.f);
      }
    }
    __syncthreads();
    // ---- fc2: samples 16 warp .. +15 (two n-tiles), all 6 output tiles
    {
      uint32_t b[8][4];
      const uint32_t b_base = h1_s + (uint32_t)(((16 * warp + b_row) * kH1S + b_col) * 2);
#pragma unroll
      for (int st = 0; st < 8; ++st) ldmatrix_x4(b[st], b_base + st * 32);
#pragma unroll
      for (int mt = 0; mt < 6; ++mt) {
        float d[2][4] = {};
        const uint32_t a_base = wf2_s + (uint32_t)(((16 * mt + a_row) * kF2S + a_col) * 2);
#pragma unroll
        for (int st = 0; st < 8; ++st) {
          uint32_t a[4];
          ldmatrix_x4(a, a_base + st * 32);
          mma_bf16(d[0], a[0], a[1], a[2], a[3], b[st][0], b[st][1]);
          mma_bf16(d[1], a[0], a[1], a[2], a[3], b[st][2], b[st][3]);
        }
        const int j0 = 16 * mt + g, j1 = j0 + 8;
        const float c0 = j0 < 84 ? bf2[j0] : 0.f, c1 = j1 < 84 ? bf2[j1] : 0.f;
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          const int s0 = 16 * warp + 8 * n + 2 * c;
          h2[s0 * kH2S + j0] = __float2bfloat16(j0 < 84 ? fmaxf(d[n][0] + c0, 0.f) : 0.f);
          h2[(s0 + 1) * kH2S + j0] = __float2bfloat16(j0 < 84 ? fmaxf(d[n][1] + c0, 0.f) : 0.f);
          h2[s0 * kH2S + j1] = __float2bfloat16(j1 < 84 ? fmaxf(d[n][2] + c1, 0.f) : 0.f);
          h2[(s0 + 1) * kH2S + j1] = __float2bfloat16(j1 < 84 ? fmaxf(d[n][3] + c1, 0.f) : 0.f);
        }
      }
    }
    // fc3 reads only this warp's own h2 rows (samples 16 warp .. +15)
    __syncwarp();
    float loss;
    {
      float d[2][4] = {};
      const uint32_t b_base = h2_s + (uint32_t)(((16 * warp + b_row) * kH2S + b_col) * 2);
      const uint32_t a_base = wf3_s + (uint32_t)((a_row * kF3S + a_col) * 2);
#pragma unroll
      for (int st = 0; st < 6; ++st) {
        uint32_t a[4], b[4];
        ldmatrix_x4(a, a_base + st * 32);
        ldmatrix_x4(b, b_base + st * 32);
        mma_bf16(d[0], a[0], a[1], a[2], a[3], b[0], b[1]);
        mma_bf16(d[1], a[0], a[1], a[2], a[3], b[2], b[3]);
      }
      // logits[sample][class]; h1 is dead once every warp has passed fc2
      __syncthreads();
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        const int s0 = 16 * warp + 8 * n + 2 * c;
        logit[s0 * 16 + g] = d[n][0] + bf3[g];
        logit[(s0 + 1) * 16 + g] = d[n][1] + bf3[g];
        if (g < 2) {
          logit[s0 * 16 + g + 8] = d[n][2] + bf3[g + 8];
          logit[(s0 + 1) * 16 + g + 8] = d[n][3] + bf3[g + 8];
        }
      }
      __syncwarp();
      loss = 0.f;
      const uint32_t s = s_lo + 16 * warp + lane;
      if (lane < 16 && s < s_hi) {
        const float* z = logit + (16 * warp + lane) * 16;
        float m = z[0];
#pragma unroll
        for (int q = 1; q < 10; ++q) m = fmaxf(m, z[q]);
        float se = 0.f;
#pragma unroll
        for (int q = 0; q < 10; ++q) se += expf(z[q] - m);
        loss = (m + logf(se)) - z[args.y[s]];
      }
    }
    // fixed-order reduction: 16 lanes per warp, then the 8 warps in order
    loss += __shfl_xor_sync(0xffffffffu, loss, 1);
    loss += __shfl_xor_sync(0xffffffffu, loss, 2);
    loss += __shfl_xor_sync(0xffffffffu, loss, 4);
    loss += __shfl_xor_sync(0xffffffffu, loss, 8);
    if (lane == 0) wsum[warp] = loss;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int w = 0; w < kFcWarps; ++w) t += wsum[w];
      args.part[(row * args.nparts + part) * 2] = t;
      args.part[(row * args.nparts + part) * 2 + 1] = 0.0f;
    }
  }
}

// ============================================================ fused kernel
// k_lenet_fused — conv (warp-level MMA, as k_lenet_conv) and the fc stack on
// the 5th-gen tensor cores in one CTA per SM, with no activation scratch in
// HBM.  Work item = (candidate, 128-sample chunk):
//   1. conv: 8 warps, one sample each at a time (conv1_pairs + conv2_tiles);
//      each sample's pooled conv2 output (400 bf16) goes straight into the
//      fc1 A operand in shared memory (tcgen05 no-swizzle K-major layout,
//      K = channel * 25 + window, the natural f1w column order);
//   2. fc1 = tcgen05.mma kind::f16 M = 128 samples, N = 128 (120 outputs),
//      K = 400 with A and B (f1w, staged from the candidate row in two
//      K halves through the conv buffers) in shared memory, D1 in TMEM;
//   3. +b1, ReLU, bf16 -> back into TMEM (tcgen05.st) as the A operand of
//      fc2 (M = 128, N = 96 (84), K = 128 (120), B = f2w in shared memory),
//      the same for fc3 (N = 16 (10), K = 96 (84)) — MMAs with A in TMEM;
//   4. logits (tcgen05.ld, one sample per thread) -> CE -> fixed-order sums.
// TMEM columns: A2 [0, 64), A3 [64, 112), D1 [256, 384), D2 [384, 480),
// D3 [480, 496) of a 512-column allocation.
namespace {

constexpr int kFW = 8;  // conv warps (smem: 8 x (pair image + pooled map) + the fc1 A operand)
constexpr int kFThreads = kFW * 32;

// byte offset of element (r, k) in a no-swizzle K-major tcgen05 operand of
// R rows: 8-row x 16-byte core matrices, LBO (along K) = R * 16, SBO = 128
__host__ __device__ constexpr uint32_t il_off(uint32_t r, uint32_t k, uint32_t R) {
  return (k >> 3) * (R * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

struct FusedSmem {
  static constexpr int wc1 = 0;                                // [8][32] bf16
  static constexpr int wc2 = wc1 + 8 * kC1K * 2;               // [16][216] bf16
  static constexpr int bc1 = wc2 + 16 * kC2S * 2;              // f32 [8]
  static constexpr int bc2 = bc1 + 8 * 4;                      // f32 [16]
  static constexpr int img = (bc2 + 16 * 4 + 127) / 128 * 128;  // per warp [33][40] u32 | f1w half (TMA dst)
  static constexpr int p1 = img + kFW * kImgWords * 4;         // per warp [14][kP1R][4] u32
  static constexpr int a1 = p1 + kFW * kP1Words * 4;           // fc1 A: 128 x 400 bf16
  static constexpr int w2 = a1 + 128 * 400 * 2;                // fc2 B: 96 x 128 bf16
  static constexpr int w3 = w2 + 96 * 128 * 2;                 // fc3 B: 16 x 96 bf16
  static constexpr int b1 = w3 + 16 * 96 * 2;                  // f32 [128]
  static constexpr int b2 = b1 + 128 * 4;                      // f32 [96]
  static constexpr int b3 = b2 + 96 * 4;                       // f32 [16]
  static constexpr int red = b3 + 16 * 4;                      // f32 [8]
  static constexpr int bar = red + 8 * 4;                      // u64 mbarriers: MMA commit, TMA
  static constexpr int slot = bar + 16;                        // TMEM base
  static constexpr int total = slot + 16;
};
constexpr int kF1Half0 = 208, kF1Half1 = 192;  // K per f1w half (13 + 12 MMA k-steps)
static_assert(FusedSmem::total <= 227 * 1024, "fused LeNet shared memory");
static_assert(FusedSmem::img % 16 == 0 && FusedSmem::a1 % 16 == 0 && FusedSmem::w2 % 16 == 0 &&
                  FusedSmem::w3 % 16 == 0 && FusedSmem::bar % 8 == 0, "aligned operands");
static_assert(128 * 208 * 2 <= FusedSmem::a1 - FusedSmem::img, "an f1w half fits the conv buffers");

constexpr uint32_t kColA2 = 0, kColA3 = 64, kColD1 = 256, kColD2 = 384, kColD3 = 480;

// 16 bytes = parameters [k0, k0 + 8) of row `j` (8-byte aligned source), 0 past `kmax`
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

#ifndef LENET_PROBE
#define LENET_PROBE 0  // 1: profiling probe, conv only (fc stage skipped, partials 0)
#endif

__device__ __forceinline__ void async_smem_fence() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace

// tmap_f1: 3-D view (k + 4, j, candidate) of every candidate's f1w block,
// based 4 parameters before it (the block starts 8 bytes off a 16-byte
// boundary); a box (8, 128, 1) = one 16-byte K chunk of the 128 (120 + 8
// zero-filled) rows, which lands in shared memory as one 2048-byte column of
// core matrices of the no-swizzle operand layout.
__global__ void __launch_bounds__(kFThreads, 1) k_lenet_fused(LenetArgs args,
                                                              const __grid_constant__ CUtensorMap tmap_f1) {
  using namespace tc;
  pdl_enter();
  if (args.gate != nullptr && *args.gate == 0) return;
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int wi = g >> 1, dx = g & 1;
  __nv_bfloat16* wc1 = reinterpret_cast<__nv_bfloat16*>(sm + FusedSmem::wc1);
  __nv_bfloat16* wc2 = reinterpret_cast<__nv_bfloat16*>(sm + FusedSmem::wc2);
  float* bc1 = reinterpret_cast<float*>(sm + FusedSmem::bc1);
  float* bc2 = reinterpret_cast<float*>(sm + FusedSmem::bc2);
  const uint32_t* img = reinterpret_cast<const uint32_t*>(sm + FusedSmem::img) + warp * kImgWords;
  const uint32_t img_s = smem_addr(img);
  uint32_t* p1 = reinterpret_cast<uint32_t*>(sm + FusedSmem::p1) + warp * kP1Words;
  __nv_bfloat16* a1 = reinterpret_cast<__nv_bfloat16*>(sm + FusedSmem::a1);
  float* sb1 = reinterpret_cast<float*>(sm + FusedSmem::b1);
  float* sb2 = reinterpret_cast<float*>(sm + FusedSmem::b2);
  float* sb3 = reinterpret_cast<float*>(sm + FusedSmem::b3);
  float* red = reinterpret_cast<float*>(sm + FusedSmem::red);
  const uint32_t bar = smem_u32(sm + FusedSmem::bar), bar_tma = bar + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + FusedSmem::slot);
  {
    uint32_t* p = reinterpret_cast<uint32_t*>(sm);
    for (int i = threadIdx.x; i < FusedSmem::bar / 4; i += kFThreads) p[i] = 0u;
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar_tma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_f1)));
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int q = warp & 3, hf = warp >> 2;           // TMEM lane quarter, column half
  const uint32_t lanes = tmem + ((uint32_t)(q * 32) << 16);
  const uint32_t r_s = smem_u32(sm + FusedSmem::img), a1_s = smem_u32(a1);
  const uint32_t w2_s = smem_u32(sm + FusedSmem::w2), w3_s = smem_u32(sm + FusedSmem::w3);
  uint32_t phase = 0, tphase = 0;
  auto mma_round = [&]() {  // every thread: wait for the MMAs committed to `bar`
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
  };

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
      // fc2 / fc3 B operands (rows past 84 / 10 and K past 120 / 84 are zero) and biases
      for (int i = threadIdx.x; i < 96 * 16; i += kFThreads) {
        const int j = i / 16, cc = i - 16 * j;
        const uint4 v = j < 84 ? load8(w + oF2W + j * 120, 8 * cc, 120) : make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(sm + FusedSmem::w2 + il_off(j, 8 * cc, 96)) = v;
      }
      for (int i = threadIdx.x; i < 16 * 12; i += kFThreads) {
        const int j = i / 12, cc = i - 12 * j;
        const uint4 v = j < 10 ? load8(w + oF3W + j * 84, 8 * cc, 84) : make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(sm + FusedSmem::w3 + il_off(j, 8 * cc, 16)) = v;
      }
      if (threadIdx.x < 128) sb1[threadIdx.x] = threadIdx.x < 120 ? bf(w[oF1B + threadIdx.x]) : 0.f;
      if (threadIdx.x < 96) sb2[threadIdx.x] = threadIdx.x < 84 ? bf(w[oF2B + threadIdx.x]) : 0.f;
      if (threadIdx.x < 16) sb3[threadIdx.x] = threadIdx.x < 10 ? bf(w[oF3B + threadIdx.x]) : 0.f;
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
    // ---- 1. conv for the chunk's samples -> fc1 A operand
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
    // ---- 2. fc1: D1 = A1 (128 x 400) . f1w^T, two K halves of f1w through the conv buffers
    uint32_t kk0 = 0;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int k0 = h == 0 ? 0 : kF1Half0, kh = h == 0 ? kF1Half0 : kF1Half1;
      if (threadIdx.x == 0) {  // TMA: one 2048-byte K chunk of f1w per box
        mbar_expect_tx(bar_tma, (uint32_t)kh / 8 * 2048);
        for (int cc = 0; cc < kh / 8; ++cc)
          tma_load_3d(r_s + cc * 2048, &tmap_f1, bar_tma, k0 + 8 * cc, 0, (int)row);
      }
      mbar_wait(bar_tma, tphase);
      tphase ^= 1;
      if (threadIdx.x == 0) {
        tc_fence_after();
        constexpr uint32_t id1 = idesc_bf16(128, 128);
        for (int kk = 0; kk < kh / 16; ++kk) {
          const uint64_t da = interleaved_desc(a1_s + (kk0 + kk) * 2 * 2048, 2048, 128);
          const uint64_t db = interleaved_desc(r_s + kk * 2 * 2048, 2048, 128);
          mma_ss(tmem + kColD1, da, db, id1, (kk0 + kk) != 0);
        }
        mma_commit(bar);
      }
      kk0 += kh / 16;
      mma_round();  // also frees the f1w half buffer
    }
    // ---- 3. fc1 epilogue -> A2, fc2, fc2 epilogue -> A3, fc3
#pragma unroll 1
    for (int cc = 0; cc < 2; ++cc) {
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
      mma_commit(bar);
    }
    mma_round();
    {
      // D2 columns [hf * 48, hf * 48 + 48): 32 + 16
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
      uint32_t pk2[16];
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
      mma_commit(bar);
    }
    mma_round();
    // ---- 4. logits -> CE (thread = sample), fixed-order sums
    float loss = 0.f;
    if (hf == 0) {
      float z[16];
      tmem_ld16(lanes + kColD3, z);
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
        const int lab = args.y[smp];
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
    if (threadIdx.x == 0) {
      const float t = ((red[0] + red[1]) + red[2]) + red[3];
      args.part[(row * args.nparts + part) * 2] = t;
      args.part[(row * args.nparts + part) * 2 + 1] = 0.0f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

struct LenetPlan {
  LenetArgs args;
  bool fused;  // k_lenet_fused (default); MGFWA_LENET_FUSED=0: conv + fc kernels through the HBM scratch
  unsigned grid_fused;
  CUtensorMap tmap_f1;
  unsigned grid_conv, grid_fc;
  uint64_t group_rows;  // candidates per conv/fc launch pair (bounds the scratch)
  uint32_t* pimg;       // owned
  __nv_bfloat16* p2;    // owned scratch [group_rows][S][400]
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
      cudaFuncSetAttribute(k_lenet_fc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           FcSmem::total) != cudaSuccess ||
      cudaFuncSetAttribute(k_lenet_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           FusedSmem::total) != cudaSuccess) {
    snprintf(err, errlen, "LeNet objective: shared memory opt-in failed");
    return nullptr;
  }
  auto* p = new (std::nothrow) LenetPlan{};
  if (!p) return nullptr;
  if (cudaMalloc(&p->pimg, (size_t)S * kImgWords * 4) != cudaSuccess) {
    snprintf(err, errlen, "LeNet objective: cudaMalloc of the pair images failed");
    delete p;
    return nullptr;
  }
  const uint64_t n = (uint64_t)S * kImgWords;
  k_lenet_pairs<<<(unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256>>>(X, S, p->pimg);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    snprintf(err, errlen, "LeNet objective: pair-image kernel failed");
    cudaFree(p->pimg);
    delete p;
    return nullptr;
  }
  p->args.pimg = p->pimg;
  p->args.y = y;
  p->args.W = W;
  p->args.rows = rows;
  p->args.Dp = Dp;
  p->args.S = S;
  p->args.nparts = lenet_num_parts(S);
  {
    const char* e = getenv("MGFWA_LENET_FUSED");
    p->fused = !(e && e[0] == '0');
  }
  if (p->fused) {
    tc::EncodeTiledFn enc = tc::get_encode_fn();
    cuuint64_t dims[3] = {404, 120, rows};
    cuuint64_t strides[2] = {800, Dp * 2};
    cuuint32_t box[3] = {8, 128, 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (!enc || enc(&p->tmap_f1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<__nv_bfloat16*>(W + oF1W - 4),
                    dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      snprintf(err, errlen, "LeNet objective: f1w tensor map encode failed");
      cudaFree(p->pimg);
      delete p;
      return nullptr;
    }
    const uint64_t items = rows * p->args.nparts;
    p->grid_fused = (unsigned)(items < (uint64_t)nsm ? items : (uint64_t)nsm);
    return p;
  }
  // scratch of at most kScratchBytes (at least one candidate's activations)
  const uint64_t per_row = (uint64_t)S * kP2Row * 2;
  uint64_t cap = kScratchBytes;
  if (const char* e = getenv("MGFWA_LENET_SCRATCH_MB"))  // tests: force candidate groups
    cap = (uint64_t)strtoull(e, nullptr, 10) << 20;
  p->group_rows = cap / per_row;
  if (p->group_rows < 1) p->group_rows = 1;
  if (p->group_rows > rows) p->group_rows = rows;
  if (cudaMalloc(&p->p2, p->group_rows * per_row) != cudaSuccess) {
    snprintf(err, errlen, "LeNet objective: cudaMalloc of the activation scratch failed");
    cudaFree(p->pimg);
    delete p;
    return nullptr;
  }
  p->args.pimg = p->pimg;
  p->args.y = y;
  p->args.W = W;
  p->args.rows = rows;
  p->args.Dp = Dp;
  p->args.S = S;
  p->args.nparts = lenet_num_parts(S);
  const uint64_t items = p->group_rows * p->args.nparts;
  p->grid_conv = p->grid_fc = (unsigned)(items < (uint64_t)nsm ? items : (uint64_t)nsm);
  return p;
}

void lenet_plan_destroy(LenetPlan* p) {
  if (!p) return;
  cudaFree(p->pimg);
  cudaFree(p->p2);
  delete p;
}

cudaError_t lenet_fitness_launch(const LenetPlan* p, float* part, const int* gate,
                                 cudaStream_t s) {
  if (p->fused) {
    LenetArgs a = p->args;
    a.part = part;
    a.gate = gate;
    return pdl_launch(k_lenet_fused, p->grid_fused, kFThreads, FusedSmem::total, s, a, p->tmap_f1);
  }
  for (uint64_t r0 = 0; r0 < p->args.rows; r0 += p->group_rows) {
    LenetSplitArgs sa{p->args, p->p2};
    sa.base.W += r0 * p->args.Dp;
    sa.base.rows = p->args.rows - r0 < p->group_rows ? p->args.rows - r0 : p->group_rows;
    sa.base.part = part + r0 * p->args.nparts * 2;
    sa.base.gate = gate;
    const uint64_t items = sa.base.rows * sa.base.nparts;
    const unsigned gc = (unsigned)(items < p->grid_conv ? items : p->grid_conv);
    cudaError_t e = pdl_launch(k_lenet_conv, gc, kConvThreads, ConvSmem::total, s, sa);
    if (e != cudaSuccess) return e;
    e = pdl_launch(k_lenet_fc, gc, kFcThreads, FcSmem::total, s, sa);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace mgfwa_b200
