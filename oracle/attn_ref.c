/* TEST INFRASTRUCTURE — oracle restatement, never shipped or measured.
 *
 * fp32 CPU restatement of paged decode attention. The reference has no
 * attention arithmetic (it models decode as a bandwidth formula,
 * proj/src/cost_model.cpp:73-79, and states real kernels are out of scope,
 * SPEC.md:13-15), so this is the builder-written restatement the north star
 * asks for: for each query head h of the GQA group g = h / (Hq/Hkv),
 * o = softmax(q . K^T * scale) . V over the request's tokens in block order,
 * bf16 inputs, fp32 (here fp64-accumulated) math. Parity tolerance in the
 * tests: 1e-3 relative (north star). */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

uint16_t oracle_kv_value_bf16(uint64_t seed, int layer, int kv, int64_t token, int head, int dim);

static float bf16_to_f32(uint16_t b) {
  union { uint32_t u; float f; } x;
  x.u = (uint32_t)b << 16;
  return x.f;
}

/* Contiguous form: k, v [kv_len][hkv][d], q [hq][d] (bf16 bits); out [hq][d] fp32. */
void oracle_decode_attn(const uint16_t* q, const uint16_t* k, const uint16_t* v, int64_t kv_len, int hq,
                        int hkv, int d, float scale, float* out) {
  const int g = hq / hkv;
  double* s = (double*)malloc(sizeof(double) * (size_t)(kv_len > 0 ? kv_len : 1));
  for (int h = 0; h < hq; ++h) {
    const int kh = h / g;
    double m = -INFINITY;
    for (int64_t t = 0; t < kv_len; ++t) {
      double acc = 0.0;
      for (int i = 0; i < d; ++i)
        acc += (double)bf16_to_f32(q[h * d + i]) * (double)bf16_to_f32(k[(t * hkv + kh) * d + i]);
      s[t] = acc * scale;
      if (s[t] > m) m = s[t];
    }
    double l = 0.0;
    for (int64_t t = 0; t < kv_len; ++t) {
      s[t] = exp(s[t] - m);
      l += s[t];
    }
    for (int i = 0; i < d; ++i) {
      double o = 0.0;
      for (int64_t t = 0; t < kv_len; ++t) o += s[t] * (double)bf16_to_f32(v[(t * hkv + kh) * d + i]);
      out[h * d + i] = kv_len > 0 ? (float)(o / l) : 0.f;
    }
  }
  free(s);
}

/* Generator form: K/V of (layer, token, head) come from the synthetic
 * generator, so the device path (scatter, offload, prefetch, table) is
 * checked end to end. Heads [head0, head0 + hkv_local) of this shard; q
 * [hq_local][d]. */
void oracle_decode_attn_gen(uint64_t seed, int layer, int64_t kv_len, int head0, int hkv_local, int group,
                            int d, const uint16_t* q, float scale, float* out) {
  const int64_t n = kv_len * hkv_local * d;
  uint16_t* k = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(n > 0 ? n : 1));
  uint16_t* v = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t t = 0; t < kv_len; ++t)
    for (int h = 0; h < hkv_local; ++h)
      for (int i = 0; i < d; ++i) {
        k[(t * hkv_local + h) * d + i] = oracle_kv_value_bf16(seed, layer, 0, t, head0 + h, i);
        v[(t * hkv_local + h) * d + i] = oracle_kv_value_bf16(seed, layer, 1, t, head0 + h, i);
      }
  oracle_decode_attn(q, k, v, kv_len, hkv_local * group, hkv_local, d, scale, out);
  free(k);
  free(v);
}

/* Causal prefill attention (no reference arithmetic either):
 * q [tokens][hq][d], k/v [tokens][hkv][d] bf16 bits, out [tokens][hq][d] fp32;
 * query row i of head h attends keys 0..i of kv head h / (hq/hkv). */
void oracle_prefill_attn(const uint16_t* q, const uint16_t* k, const uint16_t* v, int64_t tokens, int hq,
                         int hkv, int d, float scale, float* out) {
  const int g = hq / hkv;
  double* s = (double*)malloc(sizeof(double) * (size_t)(tokens > 0 ? tokens : 1));
  double* o = (double*)malloc(sizeof(double) * (size_t)d);
  for (int64_t i = 0; i < tokens; ++i)
    for (int h = 0; h < hq; ++h) {
      const int kh = h / g;
      double m = -INFINITY;
      for (int64_t t = 0; t <= i; ++t) {
        double acc = 0.0;
        for (int e = 0; e < d; ++e)
          acc += (double)bf16_to_f32(q[(i * hq + h) * d + e]) * (double)bf16_to_f32(k[(t * hkv + kh) * d + e]);
        s[t] = acc * scale;
        if (s[t] > m) m = s[t];
      }
      double l = 0.0;
      for (int e = 0; e < d; ++e) o[e] = 0.0;
      for (int64_t t = 0; t <= i; ++t) {
        const double p = exp(s[t] - m);
        l += p;
        for (int e = 0; e < d; ++e) o[e] += p * (double)bf16_to_f32(v[(t * hkv + kh) * d + e]);
      }
      for (int e = 0; e < d; ++e) out[(i * hq + h) * d + e] = (float)(o[e] / l);
    }
  free(s);
  free(o);
}
