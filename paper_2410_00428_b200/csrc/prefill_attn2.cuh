// Causal GQA prefill attention on tcgen05: the
// per-layer compute that a layer's offload D2H hides behind
// (engine.cpp:27-31, schedule_prefill_span). The only place on the path where
// the work is a dense contraction, so the only tensor-core kernel besides the
// GQA decode tile.
//
// A CTA owns query tiles A = 2p and B = 2p + 1 of one head and gives each its
// own softmax warpgroup (thread = query row, all 128 columns), so one tile's
// exponentials overlap the other's TMEM traffic and the MMAs of the other
// tile, and every K/V tile loaded from HBM serves 256 query rows.
//
// Warps (three aligned warpgroups): 0 TMA (Q_A, Q_B, then
// the K and V rings, 2 stages each; a K stage frees when both S MMAs read it,
// a V stage when both PVs did), 1 MMA issuer + TMEM owner, 2-3 idle — this
// warpgroup drops to 56 registers with setmaxnreg — then 4-7 softmax of tile
// A and 8-11 softmax of tile B at 224 (warp w reads TMEM lanes
// 32*(w%4)..+31). (Round 1's 320-thread layout, softmax warps 2-9 at 168
// registers with a few spilled, was 2-4% slower: DESIGN.md §4.3.1.)
// TMEM (512 columns): S_A [0,128), S_B [128,256), O_A [256,384),
// O_B [384,512). P (fp16 pairs, against the fp16 copy of V) overwrites the
// first 64 columns of its S. Issue order per KV tile j:
//   ... PV_A(j-1), S_A(j), PV_B(j-1), S_B(j), PV_A(j), ...
// The tensor pipe executes in issue order, so S_A(j) never overwrites P_A(j-1)
// before PV_A(j-1) read it. P(j) is handed over in two halves (64 KV columns
// each): the PV MMAs of the first half run while the softmax computes the
// second (+1.6-1.8% at 4k-32k; four quarters lose 1%). Tile A's causal range is KV tiles 0..2p, B's is
// 0..2p+1 (the last KV tile is B's alone).
//
// P precision: bf16 P alone misses the 1e-3 bar (2^-9 per weight), so P is
// fp16 (2^-11) against an fp16 copy of V made by lkv_prefill_attention
// (bf16_to_f16_kernel; kind::f16 needs A and B in the same format). Lazy
// rescaling: the running max only moves when a tile exceeds it by more than
// 2^8; only then does the warp wait for the previous PV and rescale its O
// columns in TMEM.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "tc_sm100.cuh"

namespace lkv {

struct PrefillAttn2Smem {
  static constexpr int kStages = 2;
  static constexpr int kQ = 0;                       // Q_A, Q_B: 2 x 32 KiB
  static constexpr int kK = 65536;                   // kStages x 32 KiB
  static constexpr int kV = kK + kStages * 32768;    // kStages x 32 KiB
  static constexpr int kBar = kV + kStages * 32768;  // mbarriers
  static constexpr int kPChunks = 2;                 // P hand-offs per query tile and KV tile
  static constexpr int kNumBars = 1 + 2 * (2 + kPChunks) + 4 * kStages;
  static constexpr int kTmem = kBar + kNumBars * 8;
  static constexpr int kBytes = kTmem + 16;
  static_assert(kBytes <= 232448, "227 KiB dynamic smem limit");
};

// 2^x on the MUFU pipe, flushing denormals (-inf -> +0).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32x2 FMA / add (sm_100 FFMA2 / FADD2): half the issue slots of
// the softmax's scale-subtract and row-sum.
__device__ __forceinline__ unsigned long long f2pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(unsigned long long v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// LKV_PREFILL_TRACE (build-time, diagnostic only): clock64 stamps of CTA 0's
// softmax and MMA phases into g_pf_trace (read by lkv_debug_prefill_trace).
#ifndef LKV_PREFILL_TRACE
#define LKV_PREFILL_TRACE 0
#endif
#if LKV_PREFILL_TRACE
__device__ unsigned long long g_pf_trace[4096];
__device__ unsigned long long g_pf_cta[3 * 4096];  // per CTA: %globaltimer start, end, %smid
#define PF_TRACE(cond, idx)                                              \
  do {                                                                   \
    if (blockIdx.x == 0 && (cond) && (idx) < 4096) g_pf_trace[(idx)] = clock64(); \
  } while (0)
#else
#define PF_TRACE(cond, idx) \
  do {                      \
  } while (0)
#endif

// Register split: warpgroup 0 (TMA + MMA warps) drops to 56 registers with
// setmaxnreg, the two softmax warpgroups rise to 224 (they use 172, no
// spills); per SMSP one warp of each: (56 + 224 + 224) x 32 <= 16 K registers.
constexpr int kPrefillThreads = 384;
constexpr int kPrefillSoftmaxWarp0 = 4;  // first softmax warp
__global__ void __launch_bounds__(kPrefillThreads, 1) prefill_attn2_kernel(
    const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
    const __grid_constant__ CUtensorMap vmap, void* __restrict__ out, int out_f32, int tokens, int Hq, int G,
    float scale_log2, int chunk_q) {
  using S = PrefillAttn2Smem;
  constexpr int NS = S::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  if ((tc::saddr(sm) & 1023u) != 0u) __trap();
#if LKV_PREFILL_TRACE
  unsigned long long t_cta0 = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_cta0));
#endif
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + S::kBar);
  uint64_t* q_full = bars;
  constexpr int NC = S::kPChunks;
  uint64_t* s_full = bars + 1;  // [2] tile A, B
  uint64_t* o_full = bars + 3;  // [2]
  uint64_t* p_full = bars + 5;  // [2][NC]: P columns [128c/NC, 128(c+1)/NC) of tile t in TMEM
  uint64_t* k_full = bars + 5 + 2 * NC;  // [NS]
  uint64_t* k_empty = k_full + NS;
  uint64_t* v_full = k_empty + NS;
  uint64_t* v_empty = v_full + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + S::kTmem);

  const int nq = (tokens + 127) / 128;
  const int npairs = (nq + 1) / 2;
  // 1D grid in dispatch order: query heads in chunks of `chunk_q` (whole GQA
  // groups), and inside a chunk every head's heaviest pair first, heads
  // fastest. Within a chunk that is longest-processing-time order, so the
  // launch ends on the lightest pairs instead of a late heavy one; the chunk
  // bounds the K/V the resident CTAs stream (chunk_q / G KV heads x T x
  // 512 B) to what L2 holds, so those tiles are read from HBM about once.
  const int chunk = static_cast<int>(blockIdx.x) / (chunk_q * npairs);
  const int width = min(chunk_q, Hq - chunk * chunk_q);
  const int within = static_cast<int>(blockIdx.x) - chunk * chunk_q * npairs;
  const int pair = npairs - 1 - within / width;
  const int qa = 2 * pair, qb = 2 * pair + 1;
  const bool has_b = qb < nq;
  const int nt_a = qa + 1, nt_b = has_b ? qb + 1 : 0;
  const int nt = has_b ? nt_b : nt_a;  // KV tiles this CTA loads
  const int hq = chunk * chunk_q + within % width, h = hq / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tc::bar_init(q_full, 1);
    for (int t = 0; t < 2; ++t) {
      tc::bar_init(&s_full[t], 1);
      for (int c = 0; c < NC; ++c) tc::bar_init(&p_full[t * NC + c], 128);
      tc::bar_init(&o_full[t], 1);
    }
    for (int b = 0; b < NS; ++b) {
      tc::bar_init(&k_full[b], 1);
      tc::bar_init(&k_empty[b], 1);
      tc::bar_init(&v_full[b], 1);
      tc::bar_init(&v_empty[b], 1);
    }
    tc::bar_fence_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp < kPrefillSoftmaxWarp0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch_desc(&qmap);
      tc::tma_prefetch_desc(&kmap);
      tc::tma_prefetch_desc(&vmap);
      tc::bar_expect_tx(q_full, has_b ? 65536 : 32768);
      tc::tma_load_3d(sm + S::kQ, &qmap, 0, hq, qa * 128, q_full);
      tc::tma_load_3d(sm + S::kQ + 16384, &qmap, 64, hq, qa * 128, q_full);
      if (has_b) {
        tc::tma_load_3d(sm + S::kQ + 32768, &qmap, 0, hq, qb * 128, q_full);
        tc::tma_load_3d(sm + S::kQ + 49152, &qmap, 64, hq, qb * 128, q_full);
      }
      // K(j) then V(j): K runs a tile ahead of V in the MMA order below
      for (int j = 0; j < nt; ++j) {
        const int st = j % NS;
        const uint32_t ph = ((j / NS) & 1u) ^ 1u;
        tc::bar_wait(&k_empty[st], ph);
        tc::bar_expect_tx(&k_full[st], 32768);
        uint8_t* kt = sm + S::kK + st * 32768;
        tc::tma_load_3d(kt, &kmap, 0, h, j * 128, &k_full[st]);
        tc::tma_load_3d(kt + 16384, &kmap, 64, h, j * 128, &k_full[st]);
        tc::bar_wait(&v_empty[st], ph);
        // V is the fp16 copy the preceding kernel writes (PDL primary): wait
        // for it once, before the first V load (no-op without PDL)
        if (j == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
        tc::bar_expect_tx(&v_full[st], 32768);
        uint8_t* vt = sm + S::kV + st * 32768;
        tc::tma_load_3d(vt, &vmap, 0, h, j * 128, &v_full[st]);
        tc::tma_load_3d(vt + 16384, &vmap, 64, h, j * 128, &v_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 128, false, false);
      constexpr uint32_t idO = tc::idesc_f16(128, 128, false, true);
      const uint32_t q0 = tc::saddr(sm + S::kQ), k0 = tc::saddr(sm + S::kK), v0 = tc::saddr(sm + S::kV);
      auto qk = [&](int t, int j) {  // S_t(j) = Q_t K_j^T
        const uint32_t qt = q0 + t * 32768, kt = k0 + (j % NS) * 32768;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t o = (kk >> 2) * 16384 + (kk & 3) * 32;
          tc::mma_bf16(tmem + t * 128, tc::smem_desc(qt + o, 16, 1024, tc::kLayoutSw128),
                       tc::smem_desc(kt + o, 16, 1024, tc::kLayoutSw128), idS, kk > 0);
        }
        tc::mma_commit(&s_full[t]);
      };
      auto pv = [&](int t, int j) {  // O_t += P_t(j) V_j, each part of P as soon as it is in TMEM
        const uint32_t vt = v0 + (j % NS) * 32768;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (kk % (8 / NC) == 0) {
            tc::bar_wait(&p_full[t * NC + kk / (8 / NC)], j & 1u);
            tc::fence_after_sync();
          }
          const uint64_t bd = tc::smem_desc(vt + kk * 2048, 16384, 1024, tc::kLayoutSw128);
          tc::mma_bf16_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, bd, idO, (j > 0 || kk > 0));
        }
        tc::mma_commit(&o_full[t]);
      };
      tc::bar_wait(q_full, 0);
      for (int j = 0; j <= nt; ++j) {
        // PV of KV tile j-1 for each tile that covers it, each followed by
        // that tile's S of KV tile j (issue order = execution order)
        PF_TRACE(j < 128, 2048 + j * 8 + 3);
        if (j > 0) {
          const int jp = j - 1;
          tc::bar_wait(&v_full[jp % NS], (jp / NS) & 1u);
          tc::fence_after_sync();
        }
        PF_TRACE(j < 128, 2048 + j * 8 + 4);
        if (j < nt) {
          tc::bar_wait(&k_full[j % NS], (j / NS) & 1u);
          tc::fence_after_sync();
        }
        PF_TRACE(j < 128, 2048 + j * 8 + 0);
        if (j > 0 && j - 1 < nt_a) pv(0, j - 1);
        PF_TRACE(j < 128, 2048 + j * 8 + 1);
        if (j < nt_a) qk(0, j);
        if (j > 0 && j - 1 < nt_b) pv(1, j - 1);
        PF_TRACE(j < 128, 2048 + j * 8 + 2);
        if (j < nt_b) qk(1, j);
        if (j < nt) tc::mma_commit(&k_empty[j % NS]);
        if (j > 0) tc::mma_commit(&v_empty[(j - 1) % NS]);
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    // softmax: warpgroup t (0 = tile A, 1 = tile B), thread = query row
    const int t = (warp - kPrefillSoftmaxWarp0) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int qt = t == 0 ? qa : qb;
    const int ntt = t == 0 ? nt_a : nt_b;
    const int row = qt * 128 + r;
    const uint32_t tl = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    const uint32_t s_col = t * 128, o_col = 256 + t * 128;
    float m_run = -INFINITY, l_run = 0.f;
    float s[128];
    for (int j = 0; j < ntt; ++j) {
      tc::bar_wait(&s_full[t], j & 1u);
      // S(j) was issued after PV(j-1) by the same thread, so its commit
      // implies PV(j-1) completed: this wait returns at once. It observes
      // every o_full phase (compute-sanitizer synccheck flags a phase that
      // completes unobserved before the barrier's next arrival).
      if (j > 0) tc::bar_wait(&o_full[t], (j - 1) & 1u);
      tc::fence_after_sync();
      PF_TRACE(j < 128 && quad == 0 && lane == 0, t * 1024 + j * 8 + 0);
      const bool diag = j == qt;
      unsigned long long ls2[2] = {0ull, 0ull};  // (+0.f, +0.f) pairs
      const unsigned long long sc2 = f2pack(scale_log2, scale_log2);
      // P of S columns [32c, 32c + 32) against the reference maximum m (log2
      // units) -> fp16 pairs into TMEM over S columns [16c, 16c + 16) (already
      // in registers), their fp32 sum into ls2
      auto exps = [&](int c, float m) {
        const unsigned long long nm2 = f2pack(-m, -m);
        uint32_t ph[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float xa, xb;
          f2unpack(ffma2(f2pack(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]), sc2, nm2), xa, xb);
          const float a = ex2_approx(xa), b = ex2_approx(xb);
          ls2[i & 1] = fadd2(ls2[i & 1], f2pack(a, b));
          const __half2 h2 = __floats2half2_rn(a, b);
          ph[i] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        tc::tmem_st16(tl + s_col + c * 16, ph);
      };
      auto mask = [&](int c) {  // diagonal tile: key j*128 + col <= row
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = (c * 32 + i <= r) ? s[c * 32 + i] : -INFINITY;
      };
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      float corr = 1.f;
      bool resc = false;
      {
#pragma unroll
        for (int c = 0; c < 4; ++c) tc::tmem_ld32(tl + s_col + c * 32, s + c * 32);
        tc::tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c) tc::reg_fence<32>(s + c * 32);
        PF_TRACE(j < 128 && quad == 0 && lane == 0, t * 1024 + j * 8 + 1);
        if (diag) {
#pragma unroll
          for (int c = 0; c < 4; ++c) mask(c);
        }
#pragma unroll
        for (int c = 0; c < 128; ++c) mx[c & 3] = fmaxf(mx[c & 3], s[c]);
        const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * scale_log2;
        PF_TRACE(j < 128 && quad == 0 && lane == 0, t * 1024 + j * 8 + 2);
        if (mt > m_run + 8.f) {  // lazy rescale
          corr = (m_run == -INFINITY) ? 0.f : exp2f(m_run - mt);
          resc = j > 0;
          m_run = mt;
          l_run *= corr;
        }
        // O holds PV(j-1) (observed above) and PV(j) starts with the first
        // half of P, so a rescale happens before any exponential is handed off
        if (__any_sync(0xffffffffu, resc)) {
          const float f = resc ? corr : 1.f;
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            float o[32];
            tc::tmem_ld32(tl + o_col + c * 32, o);
            tc::tmem_wait_ld();
            tc::reg_fence<32>(o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= f;
            tc::tmem_st32(tl + o_col + c * 32, o);
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // P(j) -> TMEM over S(j), 32 columns at a time
          exps(c, m_run);
          if ((c + 1) % (4 / NC) == 0) {  // hand this part of P to the PV MMAs
            tc::tmem_wait_st();
            tc::fence_before_sync();
            tc::bar_arrive(&p_full[t * NC + c / (4 / NC)]);
          }
        }
        PF_TRACE(j < 128 && quad == 0 && lane == 0, t * 1024 + j * 8 + 3);
      }
      {
        float l0, l1, l2, l3;
        f2unpack(ls2[0], l0, l1);
        f2unpack(ls2[1], l2, l3);
        l_run += (l0 + l1) + (l2 + l3);
      }
      PF_TRACE(j < 128 && quad == 0 && lane == 0, t * 1024 + j * 8 + 4);
    }
    if (ntt > 0) {
      tc::bar_wait(&o_full[t], (ntt - 1) & 1u);
      tc::fence_after_sync();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      const long long obase = (static_cast<long long>(row) * Hq + hq) * 128;
      __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(out) + obase;
      float* dstf = static_cast<float*>(out) + obase;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float o[32];
        tc::tmem_ld32(tl + o_col + c * 32, o);
        tc::tmem_wait_ld();
        tc::reg_fence<32>(o);
        if (row < tokens && out_f32) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            *reinterpret_cast<float4*>(dstf + c * 32 + i * 4) =
                make_float4(o[4 * i] * inv, o[4 * i + 1] * inv, o[4 * i + 2] * inv, o[4 * i + 3] * inv);
        } else if (row < tokens) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            uint4 v;
            v.x = tc::pack_bf16(o[8 * i + 0] * inv, o[8 * i + 1] * inv);
            v.y = tc::pack_bf16(o[8 * i + 2] * inv, o[8 * i + 3] * inv);
            v.z = tc::pack_bf16(o[8 * i + 4] * inv, o[8 * i + 5] * inv);
            v.w = tc::pack_bf16(o[8 * i + 6] * inv, o[8 * i + 7] * inv);
            *reinterpret_cast<uint4*>(dst + c * 32 + i * 8) = v;
          }
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_free<512>(tmem);
#if LKV_PREFILL_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 4096) {
    unsigned long long t1, sm_id;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    asm volatile("{ .reg .u32 r; mov.u32 r, %%smid; cvt.u64.u32 %0, r; }" : "=l"(sm_id));
    g_pf_cta[3 * blockIdx.x] = t_cta0;
    g_pf_cta[3 * blockIdx.x + 1] = t1;
    g_pf_cta[3 * blockIdx.x + 2] = sm_id;
  }
#endif
}

}  // namespace lkv
