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
  long bad = 0, nfast = 0;
  for (long i = 0; i < n; ++i) {
    uint64_t pre = g();
    uint32_t d = (uint32_t)g();
    if (i & 1) d &= 0x3FFFF;  // the coordinate range of the configs
    if (i % 3 == 0) {  // a third of the prefixes put the chunk's Q_lo near the carry boundary
      const uint32_t qlo = 0xFFFFFE00u + (uint32_t)(g() % 4096) - 2048u;
      const uint32_t plo = (qlo - 0x7F4A7C15u) ^ (d & ~511u);
      pre = (pre & ~0xFFFFFFFFull) | plo;
    }
    const uint64_t h = splitmix64(pre ^ (uint64_t)d);
    const MixState z = mix_draw(draw_key(pre), d, 1u);
    const uint64_t zz = ((uint64_t)z.hi << 32) | z.lo;
    bad += (zz ^ (zz >> 31)) != h;
    bad += mant_lo(z) != (uint32_t)(h >> 11);
    bad += (z.hi >> 11) != (uint32_t)(h >> 43);
    // chunk-constant form (chunk_draw / chunk_slice / mix_chunk)
    const uint32_t cbase = d & ~511u, j = d & 511u;
    const ChunkDraw k = chunk_draw(pre, cbase);
    const uint64_t q = ((pre ^ cbase) & ~511ull) + 0x9E3779B97F4A7C15ull;
    if (chunk_fast(k)) {
      const uint32_t zlo = k.qe[j & 3u] + chunk_slice(k, j & ~3u);
      const MixState c = mix_chunk(k, zlo);
      bad += c.lo != z.lo || c.hi != z.hi;
      ++nfast;
    } else {
      bad += (uint32_t)q <= 0xFFFFFE00u;  // only near-carry chunks may be slow
    }
  }
  printf("%ld mismatches in %ld draws (%ld chunk-constant)\n", bad, n, nfast);
  return bad != 0;
}
