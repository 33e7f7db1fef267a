/* TEST INFRASTRUCTURE — CPU baseline (oracle port), timed by bench.py's
 * cpu_baseline leg and by `bench.py --impl reference`. Never shipped.
 *
 * The reference moves no bytes and computes no attention: it
 * only books the per-layer fetch (kv_manager.cpp:290-304) and charges a
 * bandwidth formula (cost_model.cpp:73-79). This port EXECUTES that decode
 * step on the host cores: for one layer of one request it (1) gathers the
 * request's CPU-resident slots of that layer into a contiguous arena with
 * memcpy (the prefetch the reference books), then (2) runs fp32 paged decode
 * attention over the arena for every query head — split over `threads`
 * pthreads by KV head. Same slot layout as the device: [K|V][H][bs][d] bf16. */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const uint8_t* host_pool;
  const uint32_t* slots;
  int64_t slot_bytes;
  int nblk, kv_len, hkv, group, bs, d;
  const uint16_t* q;
  float scale;
  float* out;
  uint8_t* arena;
  int t, nt;
} job_t;

static inline float bf(uint16_t b) {
  union { uint32_t u; float f; } x;
  x.u = (uint32_t)b << 16;
  return x.f;
}

static void* copy_part(void* p) {
  job_t* j = (job_t*)p;
  for (int b = j->t; b < j->nblk; b += j->nt)
    memcpy(j->arena + (int64_t)b * j->slot_bytes, j->host_pool + (int64_t)j->slots[b] * j->slot_bytes,
           (size_t)j->slot_bytes);
  return NULL;
}

static void* attn_part(void* p) {
  job_t* j = (job_t*)p;
  const int d = j->d, bs = j->bs;
  float* s = (float*)malloc(sizeof(float) * (size_t)(j->kv_len > 0 ? j->kv_len : 1));
  float acc[512];
  for (int h = j->t; h < j->hkv; h += j->nt) {
    for (int g = 0; g < j->group; ++g) {
      const int hq = h * j->group + g;
      const uint16_t* q = j->q + (int64_t)hq * d;
      float m = -INFINITY;
      for (int t = 0; t < j->kv_len; ++t) {
        const uint16_t* k = (const uint16_t*)(j->arena + (int64_t)(t / bs) * j->slot_bytes) +
                            ((int64_t)h * bs + t % bs) * d;
        float a = 0.f;
        for (int i = 0; i < d; ++i) a += bf(q[i]) * bf(k[i]);
        s[t] = a * j->scale;
        if (s[t] > m) m = s[t];
      }
      float l = 0.f;
      for (int i = 0; i < d; ++i) acc[i] = 0.f;
      for (int t = 0; t < j->kv_len; ++t) {
        const float p = expf(s[t] - m);
        l += p;
        const uint16_t* v = (const uint16_t*)(j->arena + (int64_t)(t / bs) * j->slot_bytes) +
                            ((int64_t)(j->hkv + h) * bs + t % bs) * d;
        for (int i = 0; i < d; ++i) acc[i] += p * bf(v[i]);
      }
      for (int i = 0; i < d; ++i) j->out[(int64_t)hq * d + i] = j->kv_len > 0 ? acc[i] / l : 0.f;
    }
  }
  free(s);
  return NULL;
}

static void run_parallel(void* (*fn)(void*), job_t* base, int threads) {
  pthread_t tid[256];
  job_t jobs[256];
  if (threads > 256) threads = 256;
  for (int i = 0; i < threads; ++i) {
    jobs[i] = *base;
    jobs[i].t = i;
    jobs[i].nt = threads;
    pthread_create(&tid[i], NULL, fn, &jobs[i]);
  }
  for (int i = 0; i < threads; ++i) pthread_join(tid[i], NULL);
}

/* One decode layer of one request on the CPU: gather + fp32 attention. */
void cpu_decode_layer(const uint8_t* host_pool, const uint32_t* slots, int nblk, int64_t slot_bytes, int kv_len,
                      int hkv, int group, int bs, int d, const uint16_t* q, float scale, float* out,
                      uint8_t* arena, int threads) {
  job_t j = {host_pool, slots, slot_bytes, nblk, kv_len, hkv, group, bs, d, q, scale, out, arena, 0, 1};
  run_parallel(copy_part, &j, threads);
  run_parallel(attn_part, &j, threads);
}
