// Host-side check that the split per-coordinate draw of the explode kernel
// (draw_key / mix_draw / mant_lo, csrc/common.cuh) reproduces
// splitmix64(prefix ^ d) (rng.hpp:33-38) bit for bit: the mixer state z,
// z ^ (z >> 31) == splitmix64, and the mantissa / top-bit words the unit
// draws read.  Built and run by tests/test_draw_split.py (nvcc, host code only).
#include <cstdint>
#include <cstdio>
#include <random>

#include "common.cuh"

using namespace mgfwa_b200;

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 1000000;
  std::mt19937_64 g(12345);
  long bad = 0;
  for (long i = 0; i < n; ++i) {
    const uint64_t pre = g();
    uint32_t d = (uint32_t)g();
    if (i & 1) d &= 0x3FFFF;  // the coordinate range of the configs
    const uint64_t h = splitmix64(pre ^ (uint64_t)d);
    const MixState z = mix_draw(draw_key(pre), d, 1u);
    const uint64_t zz = ((uint64_t)z.hi << 32) | z.lo;
    bad += (zz ^ (zz >> 31)) != h;
    bad += mant_lo(z) != (uint32_t)(h >> 11);
    bad += (z.hi >> 11) != (uint32_t)(h >> 43);
  }
  printf("%ld mismatches in %ld draws\n", bad, n);
  return bad != 0;
}
