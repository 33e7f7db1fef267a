// Synthetic KV values, shared by the device generator and (restated in C) by
// oracle/kvgen.c. A value is a splitmix64 draw (the reference's Rng mixer,
// proj/include/layersim/rng.hpp:34-39) of a packed (layer, kv, token, head,
// dim) index, mapped to k/128 for k in [-128, 128): every value is exact in
// bf16, so device and CPU agree bit for bit without rounding questions.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define LKV_HD __host__ __device__ __forceinline__
#else
#define LKV_HD inline
#endif

namespace lkv {

LKV_HD std::uint64_t kv_mix(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// kv: 0 = K, 1 = V. token < 2^24, head < 256, dim < 1024, layer < 256.
LKV_HD std::uint16_t kv_value_bf16(std::uint64_t seed, int layer, int kv, std::int64_t token,
                                  int head, int dim) {
  const std::uint64_t idx =
      ((((static_cast<std::uint64_t>(layer) * 2u + static_cast<std::uint64_t>(kv)) << 24 |
         static_cast<std::uint64_t>(token)) << 8 | static_cast<std::uint64_t>(head)) << 10) |
      static_cast<std::uint64_t>(dim);
  const std::uint64_t z = kv_mix(seed + (idx + 1) * 0x9e3779b97f4a7c15ull);
  const int k = static_cast<int>(static_cast<std::int8_t>(z >> 56));  // [-128, 127]
  // bf16 bits of k / 128 (exact: |k| < 256 needs <= 8 significant bits).
  if (k == 0) return 0;
  const std::uint32_t sign = k < 0 ? 0x8000u : 0u;
  std::uint32_t mag = static_cast<std::uint32_t>(k < 0 ? -k : k);
  int e = 0;  // mag in [2^e, 2^(e+1))
  while ((mag >> (e + 1)) != 0) ++e;
  // value = mag * 2^-7 = 1.f * 2^(e-7); bf16 exponent bias 127, 7 mantissa bits
  const std::uint32_t exp = static_cast<std::uint32_t>(127 + e - 7);
  const std::uint32_t frac = (mag << (7 - e)) & 0x7Fu;
  return static_cast<std::uint16_t>(sign | (exp << 7) | frac);
}

// Query values: same mixer on a disjoint index space (kv = 2 tag).
LKV_HD std::uint16_t q_value_bf16(std::uint64_t seed, int layer, std::int64_t seq, int qhead,
                                 int dim) {
  return kv_value_bf16(seed ^ 0x51ed2701f00dull, layer, 0, seq, qhead, dim);
}

}  // namespace lkv
