// Causal GQA prefill attention on tcgen05: the
// per-layer compute that a layer's offload D2H hides behind
// (engine.cpp:27-31, schedule_prefill_span). The only place on the path where
// the work is a dense contraction, so the only tensor-core kernel besides the
// GQA decode tile.
//
// A CTA owns query tiles A = 2p and B = 2p + 1 of one head and gives each its
// own softmax warpgroup (thread = query row, all 128 columns), so one tile's
// exponentials overlap the other tile's MMAs, and every K/V tile loaded from
// HBM serves 256 query rows.
//
// Warpgroups (384 threads; setmaxnreg moves registers to the softmax):
//   WG0  warp 0 TMA (Q_A, Q_B, then the K and V rings, 2 stages each; a K
//        stage frees when both S MMAs read it, a V stage when both PVs did),
//        warp 1 MMA issuer + TMEM owner, warps 2-3 idle; 56 registers;
//   WG1  softmax of tile A, WG2 softmax of tile B (warp w reads TMEM lanes
//        32*(w%4)..+31); 224 registers.
// TMEM (512 columns): S_A [0,128), S_B [128,256), O_A [256,384),
// O_B [384,512). P (fp16 pairs, against the fp16 copy of V) overwrites the
// first 64 columns of its S. Issue order per KV tile j:
//   ... PV_A(j-1), S_A(j), PV_B(j-1), S_B(j), PV_A(j), ...
// The tensor pipe executes in issue order, so S_A(j) never overwrites P_A(j-1)
// before PV_A(j-1) read it. Tile A's causal range is KV tiles 0..2p, B's is
// 0..2p+1 (the last KV tile is B's alone).
//
// The softmax of one tile must fit in the other tile's PV + S MMA time
// (~1000 cycles) for the tensor pipe to stay busy, and 128 exponentials per
// row on the MUFU alone take that long. So:
//   - exponentials are speculative: taken against the running max before
//     the tile's max is known (the max is folded in on the ALU pipe while
//     the MUFU works); only when a row's tile max exceeds the running max by
//     more than 2^8 (lazy rescale) does the warp recompute the tile's P
//     against the new max and rescale its O columns in TMEM;
//   - S is read from TMEM in four 32-column chunks, each load in flight
//     while the previous chunk is exponentiated, and each chunk's P is
//     stored as soon as it exists;
//   - POLY of every 4 column pairs take 2^x on the FMA pipe (ex2_poly2).
//
// P precision: bf16 P alone misses the 1e-3 bar (2^-9 per weight), so P is
// fp16 (2^-11) against an fp16 copy of V made by lkv_prefill_attention
// (bf16_to_f16_kernel; kind::f16 needs A and B in the same format).
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
  static constexpr int kNumBars = 2 + 2 * 4 + 4 * kStages;
  static constexpr int kTmem = kBar + kNumBars * 8;
  static constexpr int kBytes = kTmem + 16;
  static_assert(kBytes <= 232448, "227 KiB dynamic smem limit");
};

constexpr int kPrefillThreads = 384;

// 2^x on the MUFU pipe, flushing denormals (-inf -> +0).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32x2 FMA / add (sm_100 FFMA2 / FADD2): half the issue slots.
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

// 2^x for a pair on the FMA/ALU pipes (x <= ~126): round-to-nearest split
// x = n + f with the 1.5*2^23 trick, a degree-3 fit of 2^f on [-0.5, 0.5]
// (max relative error 1.03e-4, below fp16 P's 2^-11 rounding), n added to
// the exponent field. x = -inf (masked) clamps to 2^-127 -> 0 in fp16.
// ~10 issue slots per pair, none on the MUFU.
__device__ __forceinline__ void ex2_poly2(float xa, float xb, float& pa, float& pb) {
  const unsigned long long magic = f2pack(12582912.f, 12582912.f), neg_magic = f2pack(-12582912.f, -12582912.f);
  const unsigned long long m1 = f2pack(-1.f, -1.f), one = f2pack(1.f, 1.f);
  const unsigned long long c3 = f2pack(0.05500683f, 0.05500683f), c2 = f2pack(0.2422056f, 0.2422056f),
                           c1 = f2pack(0.69328254f, 0.69328254f);
  const unsigned long long x = f2pack(fmaxf(xa, -127.f), fmaxf(xb, -127.f));
  const unsigned long long t = fadd2(x, magic);      // 1.5*2^23 + n, n = rint(x)
  const unsigned long long r = fadd2(t, neg_magic);  // n
  const unsigned long long f = ffma2(r, m1, x);      // x - n in [-0.5, 0.5]
  const unsigned long long p = ffma2(ffma2(ffma2(c3, f, c2), f, c1), f, one);
  float ta, tb, qa, qb;
  f2unpack(t, ta, tb);
  f2unpack(p, qa, qb);
  // (t_bits << 23) == n << 23 mod 2^32: the magic's bits shift out
  pa = __int_as_float(__float_as_int(qa) + (__float_as_int(ta) << 23));
  pb = __int_as_float(__float_as_int(qb) + (__float_as_int(tb) << 23));
}

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 h2 = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h2);
}

// POLY: of every 4 column pairs, this many use ex2_poly2 (0, 1 or 2).
template <int POLY>
__global__ void __launch_bounds__(kPrefillThreads, 1) prefill_attn2_kernel(
    const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
    const __grid_constant__ CUtensorMap vmap, void* __restrict__ out, int out_f32, int tokens, int Hq, int G,
    float scale_log2, int chunk_q) {
  using S = PrefillAttn2Smem;
  constexpr int NS = S::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  if ((tc::saddr(sm) & 1023u) != 0u) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + S::kBar);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 1;  // Q buffers free: the item's last S MMA completed
  uint64_t* s_full = bars + 2;   // [2] tile A, B
  uint64_t* p_full = bars + 4;   // [2]
  uint64_t* o_full = bars + 6;   // [2]
  uint64_t* o_empty = bars + 8;  // [2] the softmax read its O out (epilogue done)
  uint64_t* k_full = bars + 10;  // [NS]
  uint64_t* k_empty = k_full + NS;
  uint64_t* v_full = k_empty + NS;
  uint64_t* v_empty = v_full + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + S::kTmem);

  const int nq = (tokens + 127) / 128;
  const int npairs = (nq + 1) / 2;
  const int n_items = npairs * Hq;
  // Work item = (query head, pair of query tiles). Items are numbered in
  // dispatch order: query heads in chunks of `chunk_q` (whole GQA groups),
  // and inside a chunk every head's heaviest pair first, heads fastest —
  // longest-processing-time order, so the launch ends on the lightest pairs;
  // the chunk bounds the K/V the resident CTAs stream (chunk_q / G KV heads x
  // T x 512 B) to what L2 holds, so those tiles are read from HBM about once.
  // A CTA takes items blockIdx.x, + gridDim.x, ... (persistent when the grid
  // is one CTA per SM: the next item's Q load and first S MMAs overlap this
  // item's epilogue, and TMEM / barrier setup is paid once).
  struct Item {
    int hq, h, qa, qb, nt_a, nt_b, nt;
  };
  auto item_of = [&](int it) {
    Item x;
    const int chunk = it / (chunk_q * npairs);
    const int width = min(chunk_q, Hq - chunk * chunk_q);
    const int within = it - chunk * chunk_q * npairs;
    const int pair = npairs - 1 - within / width;
    x.qa = 2 * pair;
    x.qb = 2 * pair + 1;
    const bool has_b = x.qb < nq;
    x.nt_a = x.qa + 1;
    x.nt_b = has_b ? x.qb + 1 : 0;
    x.nt = has_b ? x.nt_b : x.nt_a;  // KV tiles the item loads
    x.hq = chunk * chunk_q + within % width;
    x.h = x.hq / G;
    return x;
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wg = warp >> 2;

  if (threadIdx.x == 0) {
    tc::bar_init(q_full, 1);
    tc::bar_init(q_empty, 1);
    for (int t = 0; t < 2; ++t) {
      tc::bar_init(&s_full[t], 1);
      tc::bar_init(&p_full[t], 128);
      tc::bar_init(&o_full[t], 1);
      tc::bar_init(&o_empty[t], 128);
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

  if (wg == 0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (warp == 0 && lane == 0) {
      tc::tma_prefetch_desc(&qmap);
      tc::tma_prefetch_desc(&kmap);
      tc::tma_prefetch_desc(&vmap);
      int g = 0;  // KV tiles loaded so far (ring position)
      int n = 0;  // items so far
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++n) {
        const Item x = item_of(it);
        const bool has_b = x.nt_b > 0;
        if (n > 0) tc::bar_wait(q_empty, (n - 1) & 1u);  // the previous item's S MMAs read Q
        tc::bar_expect_tx(q_full, has_b ? 65536 : 32768);
        tc::tma_load_3d(sm + S::kQ, &qmap, 0, x.hq, x.qa * 128, q_full);
        tc::tma_load_3d(sm + S::kQ + 16384, &qmap, 64, x.hq, x.qa * 128, q_full);
        if (has_b) {
          tc::tma_load_3d(sm + S::kQ + 32768, &qmap, 0, x.hq, x.qb * 128, q_full);
          tc::tma_load_3d(sm + S::kQ + 49152, &qmap, 64, x.hq, x.qb * 128, q_full);
        }
        // K(j) then V(j): K runs a tile ahead of V in the MMA order below
        for (int j = 0; j < x.nt; ++j, ++g) {
          const int st = g % NS;
          const uint32_t ph = ((g / NS) & 1u) ^ 1u;
          tc::bar_wait(&k_empty[st], ph);
          tc::bar_expect_tx(&k_full[st], 32768);
          uint8_t* kt = sm + S::kK + st * 32768;
          tc::tma_load_3d(kt, &kmap, 0, x.h, j * 128, &k_full[st]);
          tc::tma_load_3d(kt + 16384, &kmap, 64, x.h, j * 128, &k_full[st]);
          tc::bar_wait(&v_empty[st], ph);
          // V is the fp16 copy the preceding kernel writes (PDL primary): wait
          // for it once, before the first V load (no-op without PDL)
          if (g == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
          tc::bar_expect_tx(&v_full[st], 32768);
          uint8_t* vt = sm + S::kV + st * 32768;
          tc::tma_load_3d(vt, &vmap, 0, x.h, j * 128, &v_full[st]);
          tc::tma_load_3d(vt + 16384, &vmap, 64, x.h, j * 128, &v_full[st]);
        }
      }
    } else if (warp == 1 && lane == 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 128, false, false);
      constexpr uint32_t idO = tc::idesc_f16(128, 128, false, true);
      const uint32_t q0 = tc::saddr(sm + S::kQ), k0 = tc::saddr(sm + S::kK), v0 = tc::saddr(sm + S::kV);
      int g = 0;                     // KV tiles consumed so far (ring position)
      int np[2] = {0, 0};            // P tiles consumed per query tile (p_full phase)
      int ne[2] = {0, 0};            // items with work per query tile (o_empty phase)
      auto qk = [&](int t, int gj) {  // S_t = Q_t K^T (KV tile at ring position gj)
        const uint32_t qt = q0 + t * 32768, kt = k0 + (gj % NS) * 32768;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t o = (kk >> 2) * 16384 + (kk & 3) * 32;
          tc::mma_bf16(tmem + t * 128, tc::smem_desc(qt + o, 16, 1024, tc::kLayoutSw128),
                       tc::smem_desc(kt + o, 16, 1024, tc::kLayoutSw128), idS, kk > 0);
        }
        tc::mma_commit(&s_full[t]);
      };
      auto pv = [&](int t, int gj, bool first) {  // O_t (+)= P_t V
        // the item's first PV overwrites O_t: the previous item's epilogue
        // must have read it out (its S MMAs ran meanwhile)
        if (first && ne[t] > 0) tc::bar_wait(&o_empty[t], (ne[t] - 1) & 1u);
        tc::bar_wait(&p_full[t], np[t] & 1u);
        ++np[t];
        tc::fence_after_sync();
        const uint32_t vt = v0 + (gj % NS) * 32768;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = tc::smem_desc(vt + kk * 2048, 16384, 1024, tc::kLayoutSw128);
          tc::mma_bf16_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, bd, idO, (!first || kk > 0));
        }
        tc::mma_commit(&o_full[t]);
      };
      int n = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++n) {
        const Item x = item_of(it);
        tc::bar_wait(q_full, n & 1u);
        tc::fence_after_sync();
        for (int j = 0; j <= x.nt; ++j) {
          // PV of KV tile j-1 for each tile that covers it, each followed by
          // that tile's S of KV tile j (issue order = execution order)
          if (j > 0) {
            const int gp = g + j - 1;
            tc::bar_wait(&v_full[gp % NS], (gp / NS) & 1u);
            tc::fence_after_sync();
          }
          if (j < x.nt) {
            tc::bar_wait(&k_full[(g + j) % NS], ((g + j) / NS) & 1u);
            tc::fence_after_sync();
          }
          if (j > 0 && j - 1 < x.nt_a) pv(0, g + j - 1, j == 1);
          if (j < x.nt_a) qk(0, g + j);
          if (j > 0 && j - 1 < x.nt_b) pv(1, g + j - 1, j == 1);
          if (j < x.nt_b) qk(1, g + j);
          if (j == x.nt - 1) tc::mma_commit(q_empty);  // every S MMA of the item issued: Q frees at completion
          if (j < x.nt) tc::mma_commit(&k_empty[(g + j) % NS]);
          if (j > 0) tc::mma_commit(&v_empty[(g + j - 1) % NS]);
        }
        g += x.nt;
        for (int t = 0; t < 2; ++t) ne[t] += (t == 0 ? x.nt_a : x.nt_b) > 0;
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    // softmax: warpgroup 1 = tile A, 2 = tile B; thread = query row
    const int t = wg - 1;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t tl = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    const uint32_t s_col = t * 128, o_col = 256 + t * 128;
    const unsigned long long sc2 = f2pack(scale_log2, scale_log2);
    float s[128];
    // P of columns [32c, 32c + 32) against the reference maximum m (log2
    // units): fp16 pairs into ph (stored to TMEM right after: STTM reads its
    // registers at issue), their fp32 sum into ls2
    auto exps = [&](int c, float m, unsigned long long* ls2, uint32_t* ph) {
      const unsigned long long nm2 = f2pack(-m, -m);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float xa, xb, a, b;
        f2unpack(ffma2(f2pack(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]), sc2, nm2), xa, xb);
        if ((i & 3) >= 4 - POLY) {
          ex2_poly2(xa, xb, a, b);
        } else {
          a = ex2_approx(xa);
          b = ex2_approx(xb);
        }
        ls2[i & 1] = fadd2(ls2[i & 1], f2pack(a, b));
        ph[i] = pack_h2(a, b);
      }
    };
    auto mask = [&](int c) {  // diagonal tile: key j*128 + col <= row
#pragma unroll
      for (int i = 0; i < 32; ++i) s[c * 32 + i] = (c * 32 + i <= r) ? s[c * 32 + i] : -INFINITY;
    };
    int ns = 0;  // S tiles consumed (s_full phase)
    int no = 0;  // PVs committed before this item (o_full phase)
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const Item x = item_of(it);
      const int qt = t == 0 ? x.qa : x.qb;
      const int ntt = t == 0 ? x.nt_a : x.nt_b;
      if (ntt == 0) continue;
      const int row = qt * 128 + r;
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < ntt; ++j, ++ns) {
        tc::bar_wait(&s_full[t], ns & 1u);
        tc::fence_after_sync();
        const bool diag = j == qt;
        unsigned long long ls2[2] = {0ull, 0ull};  // (+0.f, +0.f) pairs
        bool resc = false;
        float corr = 1.f;
        if (j == 0) {  // no running max yet: the tile's max first
#pragma unroll
          for (int c = 0; c < 4; ++c) tc::tmem_ld32(tl + s_col + c * 32, s + c * 32);
          tc::tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 4; ++c) tc::reg_fence<32>(s + c * 32);
          if (diag) {
#pragma unroll
            for (int c = 0; c < 4; ++c) mask(c);
          }
          float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = 0; c < 128; c += 2) mx[(c >> 1) & 3] = fmaxf(mx[(c >> 1) & 3], fmaxf(s[c], s[c + 1]));
          m_run = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * scale_log2;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t ph[16];
            exps(c, m_run, ls2, ph);
            tc::tmem_st16(tl + s_col + c * 16, ph);
          }
        } else {
          // speculative: exponentials against the running max while the
          // chunk loads stream in and the tile max accumulates beside them
          float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
          tc::tmem_ld32(tl + s_col, s);
          tc::tmem_wait_ld();
          tc::reg_fence<32>(s);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (c < 3) tc::tmem_ld32(tl + s_col + (c + 1) * 32, s + (c + 1) * 32);
            if (diag) mask(c);
#pragma unroll
            for (int i = 0; i < 32; i += 2)
              mx[(i >> 1) & 3] = fmaxf(mx[(i >> 1) & 3], fmaxf(s[c * 32 + i], s[c * 32 + i + 1]));
            uint32_t ph[16];
            exps(c, m_run, ls2, ph);
            // P(c) overwrites S columns [16c, 16c + 16), already in registers
            tc::tmem_st16(tl + s_col + c * 16, ph);
            if (c < 3) {
              tc::tmem_wait_ld();
              tc::reg_fence<32>(s + (c + 1) * 32);
            }
          }
          const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * scale_log2;
          const bool raise = mt > m_run + 8.f;  // lazy rescale: a weight above 2^8 moves the reference
          if (__any_sync(0xffffffffu, raise)) {  // warp-uniform: tcgen05.st is warp-collective
            if (raise) {
              corr = exp2f(m_run - mt);
              resc = true;
              m_run = mt;
              l_run *= corr;
            }
            ls2[0] = ls2[1] = 0ull;
            tc::tmem_wait_st();  // the speculative P stores land before they are replaced
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t ph[16];
              exps(c, m_run, ls2, ph);
              tc::tmem_st16(tl + s_col + c * 16, ph);
            }
          }
        }
        {
          float l0, l1, l2, l3;
          f2unpack(ls2[0], l0, l1);
          f2unpack(ls2[1], l2, l3);
          l_run += (l0 + l1) + (l2 + l3);
        }
        if (__any_sync(0xffffffffu, resc)) {  // O must hold PV(j-1) before it is rescaled
          tc::bar_wait(&o_full[t], (no + j - 1) & 1u);
          tc::fence_after_sync();
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
        tc::tmem_wait_st();
        tc::fence_before_sync();
        tc::bar_arrive(&p_full[t]);
      }
      // epilogue: O / l -> out rows, then O's columns are free for the next item
      tc::bar_wait(&o_full[t], (no + ntt - 1) & 1u);
      no += ntt;
      tc::fence_after_sync();
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      const long long obase = (static_cast<long long>(row) * Hq + x.hq) * 128;
      __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(out) + obase;
      float* dstf = static_cast<float*>(out) + obase;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float o[32];
        tc::tmem_ld32(tl + o_col + c * 32, o);
        tc::tmem_wait_ld();
        tc::reg_fence<32>(o);
        if (c == 3) {  // every O column of this thread is in registers
          tc::fence_before_sync();
          tc::bar_arrive(&o_empty[t]);
        }
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
}

}  // namespace lkv
