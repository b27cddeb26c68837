// Measures the warp-level bf16 MMA (mma.sync.m16n8k16, fp32 accumulate)
// throughput of this GPU: the ceiling of kernels that cannot use tcgen05
// (e.g. k_lenet_fitness).  Independent accumulator chains, no memory traffic.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_sync_peak mma_sync_peak.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void k(float* out) {
  float d[kChains][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
  for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 123.456f) out[0] = s;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4);
  for (int warps : {4, 8, 16, 32}) {
    const int grid = nsm * 2;
    k<<<grid, warps * 32>>>(out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<<<grid, warps * 32>>>(out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double flop = 5.0 * grid * warps * (double)kIters * kChains * 2.0 * 16 * 8 * 16;
    printf("{\"warps_per_block\": %d, \"blocks\": %d, \"tflops\": %.1f}\n", warps, grid,
           flop / (ms * 1e-3) / 1e12);
  }
  return 0;
}
