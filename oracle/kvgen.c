/* TEST INFRASTRUCTURE — oracle restatement, never shipped or measured.
 *
 * CPU restatement of the synthetic KV generator of
 * paper_2410_00428_b200/csrc/kvgen.cuh. The mixer is the reference's
 * splitmix64 (proj/include/layersim/rng.hpp:34-39); values are k/128, exact
 * in bf16. Used to check every byte the device path moves (scatter, pack,
 * D2H, H2D, gather) and to feed the attention restatement. */
#include <stdint.h>

static uint64_t mix(uint64_t z) { /* rng.hpp:35-38 */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

uint16_t oracle_kv_value_bf16(uint64_t seed, int layer, int kv, int64_t token, int head, int dim) {
  uint64_t idx = ((((uint64_t)layer * 2u + (uint64_t)kv) << 24 | (uint64_t)token) << 8 | (uint64_t)head) << 10;
  idx |= (uint64_t)dim;
  uint64_t z = mix(seed + (idx + 1) * 0x9e3779b97f4a7c15ull);
  int k = (int)(int8_t)(z >> 56);
  if (k == 0) return 0;
  uint32_t sign = k < 0 ? 0x8000u : 0u;
  uint32_t mag = (uint32_t)(k < 0 ? -k : k);
  int e = 0;
  while ((mag >> (e + 1)) != 0) ++e;
  return (uint16_t)(sign | ((uint32_t)(127 + e - 7) << 7) | ((mag << (7 - e)) & 0x7Fu));
}

uint16_t oracle_q_value_bf16(uint64_t seed, int layer, int64_t seq, int qhead, int dim) {
  return oracle_kv_value_bf16(seed ^ 0x51ed2701f00dull, layer, 0, seq, qhead, dim);
}

/* Fill [tokens][heads][dim] K and V (bf16 bits) for tokens token0.. */
void oracle_fill_kv(uint16_t* k, uint16_t* v, int64_t tokens, int64_t token0, int layer, int heads,
                    int head0, int dim, uint64_t seed) {
  for (int64_t t = 0; t < tokens; ++t)
    for (int h = 0; h < heads; ++h)
      for (int d = 0; d < dim; ++d) {
        int64_t i = (t * heads + h) * dim + d;
        k[i] = oracle_kv_value_bf16(seed, layer, 0, token0 + t, head0 + h, d);
        v[i] = oracle_kv_value_bf16(seed, layer, 1, token0 + t, head0 + h, d);
      }
}

/* Expected bytes of one (block, layer) slot in the device slot layout
 * [K|V][heads][bs][dim]; tokens >= n_tokens are zero (pack/scatter pad). */
void oracle_slot_bytes(uint16_t* out, int layer, int64_t block, int bs, int heads, int head0, int dim,
                       int64_t n_tokens, uint64_t seed) {
  for (int kv = 0; kv < 2; ++kv)
    for (int h = 0; h < heads; ++h)
      for (int t = 0; t < bs; ++t)
        for (int d = 0; d < dim; ++d) {
          int64_t tok = block * bs + t;
          out[((kv * heads + h) * bs + t) * dim + d] =
              tok < n_tokens ? oracle_kv_value_bf16(seed, layer, kv, tok, head0 + h, d) : 0;
        }
}
