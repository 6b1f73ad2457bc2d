// CounterRng (rng.hpp:12-48) on the device: splitmix64-keyed stateless
// counter RNG, bit-identical integer stream; Box-Muller with CUDA's libm
// (log / cos / sqrt), within an ulp of glibc.
#pragma once

#include <stdint.h>

namespace xbs {

__device__ __forceinline__ uint64_t mix64(uint64_t h, uint64_t v) {
  h += 0x9e3779b97f4a7c15ull + v;
  h = (h ^ (h >> 30)) * 0xbf58476d1ce4e5b9ull;
  h = (h ^ (h >> 27)) * 0x94d049bb133111ebull;
  return h ^ (h >> 31);
}
// key = mix^4(golden ^ seed, a, b, c, 0) (rng.hpp:15-19)
__device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return mix64(mix64(mix64(mix64(0x9e3779b97f4a7c15ull ^ seed, a), b), c), 0);
}
__device__ __forceinline__ double to_unit(uint64_t x) { return double(x >> 11) * 0x1.0p-53; }
// gaussian() drawing counters c0 + 1 and c0 + 2 (rng.hpp:27-33); a fresh
// generator has c0 = 0
__device__ __forceinline__ double rng_gaussian_at(uint64_t key, uint64_t c0) {
  double u1 = 1.0 - to_unit(mix64(key, c0 + 1));
  double u2 = to_unit(mix64(key, c0 + 2));
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925287 * u2);
}
__device__ __forceinline__ double rng_gaussian(uint64_t key) { return rng_gaussian_at(key, 0); }

}  // namespace xbs
