// cgm_rng.cuh -- the reference's counter-based splitmix64 streams
// (rng.cpp:12-52), Box-Muller pairs, Gray QAM points (constellation.cpp:58-66)
// and label draws, shared by the input generators (cgm_generate.cu) and the
// coded BLER harness (cgm_harness.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cgm_rng {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// Rng::fork (rng.cpp:23-25)
__host__ __device__ __forceinline__ uint64_t fork_key(uint64_t key, uint64_t stream) {
  return mix64(mix64(key ^ 0x8BB84B93962EACC9ull) + stream);
}
// Rng::next_u64 for the counter value ctr (rng.cpp:27)
__host__ __device__ __forceinline__ uint64_t draw(uint64_t key, uint64_t ctr) {
  return mix64(key + kGolden * ctr);
}
__host__ __device__ __forceinline__ double unit(uint64_t x) {
  return static_cast<double>(x >> 11) * 0x1.0p-53;
}
// One Box-Muller pair from counters (2e+1, 2e+2): (cos, sin) variates
// (rng.cpp:33-45), each scaled by sd.
__device__ __forceinline__ double2 gauss_pair(uint64_t key, uint64_t e, double sd) {
  const double u1 = 1.0 - unit(draw(key, 2 * e + 1));
  const double u2 = unit(draw(key, 2 * e + 2));
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.141592653589793 * u2;
  double sn, cs;
  sincos(angle, &sn, &cs);
  return make_double2(sd * (radius * cs), sd * (radius * sn));
}

__device__ __forceinline__ unsigned gray_decode(unsigned g) {
  unsigned m = g;
  for (unsigned s = g >> 1; s != 0; s >>= 1) m ^= s;
  return m;
}
// constellation.cpp:58-66 point of `label` in double
__device__ __forceinline__ double2 qam_point(unsigned label, int bits) {
  const int half = bits / 2;
  const unsigned levels = 1u << half;
  const double scale = 1.0 / sqrt(2.0 * ((double)levels * levels - 1.0) / 3.0);
  const unsigned gi = label >> half, gq = label & (levels - 1);
  return make_double2((2.0 * gray_decode(gi) - (levels - 1.0)) * scale,
                      (2.0 * gray_decode(gq) - (levels - 1.0)) * scale);
}
// user u's label of instance stream `key`: bits draws of next_u64() & 1 MSB first
__device__ __forceinline__ unsigned draw_label(uint64_t key, int u, int bits) {
  unsigned label = 0;
  for (int b = 0; b < bits; ++b)
    label = (label << 1) | static_cast<unsigned>(draw(key, static_cast<uint64_t>(u) * bits + b + 1) & 1u);
  return label;
}

}  // namespace cgm_rng
