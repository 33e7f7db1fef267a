// Causal GQA prefill attention on tcgen05: the
// per-layer compute that a layer's offload D2H hides behind
// (engine.cpp:27-31, schedule_prefill_span). The only place on the path where
// the work is a dense contraction, so the only tensor-core kernel besides the
// GQA decode tile.
//
// One CTA per (128-row query tile, query head), heaviest (diagonal-farthest)
// tiles first. 96 + 128*NWG threads:
//   warp 0/2   TMA producers: Q once, then K (warp 0) and V (warp 2) tiles
//              {64 d, 1 head, 128 tok} through 3D tensor maps over
//              [tokens][heads][128] (swizzle-128B, out-of-range tokens
//              zero-filled) into separate 3-stage rings. K frees at QK^T
//              completion, V at PV completion, so neither waits behind the
//              other and loads run up to two tiles ahead;
//   warp 1     MMA issuer + TMEM owner. S(j) = Q K_j^T (M=N=128, K=128) into
//              one of two TMEM S buffers; S(j+1) is issued as soon as K_{j+1}
//              lands, so QK^T overlaps the softmax of tile j. O += P_j V_j
//              accumulates in TMEM with P read from TMEM (the "TS" form: P
//              overwrites its own S buffer) and V MN-major from smem;
//   warps 3+   softmax: NWG warpgroups; thread = (query row = TMEM lane,
//              column half), its 128/NWG columns of the row in registers.
//              Lazy rescaling: the running max only moves when a tile
//              exceeds it by more than 2^8; only then does the warp wait for
//              the previous PV and rescale its O columns in TMEM.
//              P precision (bf16 P alone misses the 1e-3 bar: 2^-9 per
//              weight). PF16 (default): P in fp16 (2^-11) against an fp16
//              copy of V made by lkv_prefill_attention (every bf16 value in
//              fp16's normal range converts exactly), one PV MMA per tile.
//              !PF16: P = hi + lo in bf16, two MMAs into the same O (2^-15,
//              1.5x the MMA work); the split is integer AND/PRMT.
// TMEM: S0/P0 [0,128) S1/P1 [128,256) O [256,384) of a 512-column allocation;
// P of tile j sits in S(j)'s columns: hi [0,64), lo [64,128), two bf16 per
// column (K = token pairs), 8 columns per K=16 MMA step.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "tc_sm100.cuh"

namespace lkv {

struct PrefillAttnSmem {
  static constexpr int kStages = 3;
  static constexpr int kQ = 0;                       // 32 KiB: 2 SW128 halves (d 0-63, 64-127)
  static constexpr int kK = 32768;                   // kStages x 32 KiB
  static constexpr int kV = kK + kStages * 32768;    // kStages x 32 KiB
  static constexpr int kRed = kV + kStages * 32768;  // [2 parity][2 halves][128 rows] f32 row maxima / sums
  static constexpr int kBar = kRed + 2048;           // mbarriers
  static constexpr int kNumBars = 8 + 4 * kStages;
  static constexpr int kTmem = kBar + kNumBars * 8;
  static constexpr int kBytes = kTmem + 16;          // base is __align__(1024) (checked on entry)
  static_assert(kBytes <= 232448, "227 KiB dynamic smem limit");
};

// 2^x on the MUFU pipe, flushing denormals (-inf -> +0).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void prefill_named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// NWG softmax warpgroups split each S row by columns (NWG=2: two threads per
// query row, 64 columns each), doubling the softmax issue rate per SM; the
// halves exchange row maxima through smem once per tile.
template <int NWG, bool PF16>
__global__ void __launch_bounds__(96 + 128 * NWG, 1) prefill_attn_kernel(
    const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
    const __grid_constant__ CUtensorMap vmap, void* __restrict__ out, int out_f32, int tokens, int Hq, int G,
    float scale_log2) {
  using S = PrefillAttnSmem;
  constexpr int NS = S::kStages;
  constexpr int NSM = 128 * NWG;  // softmax threads
  constexpr int CPT = 128 / NWG;  // S columns per softmax thread
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  if ((tc::saddr(sm) & 1023u) != 0u) __trap();  // swizzle-128B tiles need 1 KiB alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + S::kBar);
  uint64_t* q_full = bars;
  uint64_t* s_full = bars + 1;    // [2] S(j) in TMEM
  uint64_t* s_empty = bars + 3;   // [2] S(j) read into registers
  uint64_t* p_full = bars + 5;    //     P(j) in TMEM
  uint64_t* o_full = bars + 6;    //     PV(j) done
  uint64_t* k_full = bars + 8;    // [NS] K ring: freed by QK^T
  uint64_t* k_empty = k_full + NS;
  uint64_t* v_full = k_empty + NS;  // [NS] V ring: freed by PV
  uint64_t* v_empty = v_full + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + S::kTmem);

  const int nq = (tokens + 127) / 128;
  const int qt = nq - 1 - static_cast<int>(blockIdx.x);
  const int hq = blockIdx.y, h = hq / G;
  const int nt = qt + 1;  // causal: KV tiles 0..qt
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tc::bar_init(q_full, 1);
    for (int b = 0; b < 2; ++b) {
      tc::bar_init(&s_full[b], 1);
      tc::bar_init(&s_empty[b], NSM);
    }
    for (int b = 0; b < NS; ++b) {
      tc::bar_init(&k_full[b], 1);
      tc::bar_init(&k_empty[b], 1);
      tc::bar_init(&v_full[b], 1);
      tc::bar_init(&v_empty[b], 1);
    }
    tc::bar_init(p_full, NSM);
    tc::bar_init(o_full, 1);
    tc::bar_fence_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch_desc(&qmap);
      tc::tma_prefetch_desc(&kmap);
      tc::bar_expect_tx(q_full, 32768);
      tc::tma_load_3d(sm + S::kQ, &qmap, 0, hq, qt * 128, q_full);
      tc::tma_load_3d(sm + S::kQ + 16384, &qmap, 64, hq, qt * 128, q_full);
      for (int j = 0; j < nt; ++j) {  // K ring: a stage frees as soon as its QK^T completes
        const int st = j % NS;
        tc::bar_wait(&k_empty[st], ((j / NS) & 1u) ^ 1u);
        tc::bar_expect_tx(&k_full[st], 32768);
        uint8_t* kt = sm + S::kK + st * 32768;
        tc::tma_load_3d(kt, &kmap, 0, h, j * 128, &k_full[st]);
        tc::tma_load_3d(kt + 16384, &kmap, 64, h, j * 128, &k_full[st]);
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {  // V ring: a stage frees when its PV completes
      tc::tma_prefetch_desc(&vmap);
      for (int j = 0; j < nt; ++j) {
        const int st = j % NS;
        tc::bar_wait(&v_empty[st], ((j / NS) & 1u) ^ 1u);
        tc::bar_expect_tx(&v_full[st], 32768);
        uint8_t* vt = sm + S::kV + st * 32768;
        tc::tma_load_3d(vt, &vmap, 0, h, j * 128, &v_full[st]);
        tc::tma_load_3d(vt + 16384, &vmap, 64, h, j * 128, &v_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 128, false, false);
      constexpr uint32_t idO = PF16 ? tc::idesc_f16(128, 128, false, true) : tc::idesc_bf16(128, 128, false, true);
      const uint32_t q0 = tc::saddr(sm + S::kQ), k0 = tc::saddr(sm + S::kK), v0 = tc::saddr(sm + S::kV);
      // PV(i) reads P(i) from S(i)'s TMEM columns; it is issued before
      // S(i+2) (same columns), and tcgen05.mma executes in issue order.
      auto pv = [&](int i) {
        const int vs = i % NS;
        tc::bar_wait(&v_full[vs], (i / NS) & 1u);
        tc::bar_wait(p_full, i & 1u);
        tc::fence_after_sync();
        const uint32_t vt = v0 + vs * 32768;
        const uint32_t pt = tmem + (i & 1) * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = tc::smem_desc(vt + kk * 2048, 16384, 1024, tc::kLayoutSw128);
          tc::mma_bf16_ts(tmem + 256, pt + kk * 8, bd, idO, (i > 0 || kk > 0));
          if constexpr (!PF16) tc::mma_bf16_ts(tmem + 256, pt + 64 + kk * 8, bd, idO, 1u);
        }
        tc::mma_commit(o_full);
        tc::mma_commit(&v_empty[vs]);
      };
      tc::bar_wait(q_full, 0);
      for (int j = 0; j < nt; ++j) {
        const int sb = j & 1, ks = j % NS;
        tc::bar_wait(&k_full[ks], (j / NS) & 1u);
        tc::bar_wait(&s_empty[sb], ((j >> 1) & 1u) ^ 1u);
        tc::fence_after_sync();
        const uint32_t kt = k0 + ks * 32768;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t o = (kk >> 2) * 16384 + (kk & 3) * 32;
          tc::mma_bf16(tmem + sb * 128, tc::smem_desc(q0 + o, 16, 1024, tc::kLayoutSw128),
                       tc::smem_desc(kt + o, 16, 1024, tc::kLayoutSw128), idS, kk > 0);
        }
        tc::mma_commit(&s_full[sb]);
        tc::mma_commit(&k_empty[ks]);
        if (j > 0) pv(j - 1);
      }
      pv(nt - 1);
    }
  } else {
    const int quad = warp & 3;
    const int wg = (warp - 3) >> 2;  // column half
    const int r = quad * 32 + lane;  // query row within the tile = TMEM lane
    const int c0 = wg * CPT;
    const int row = qt * 128 + r;
    const uint32_t tl = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    float* red = reinterpret_cast<float*>(sm + S::kRed);
    float m_run = -INFINITY, l_run = 0.f;
    float s[CPT];
    for (int j = 0; j < nt; ++j) {
      const int sb = j & 1;
      tc::bar_wait(&s_full[sb], (j >> 1) & 1u);
      tc::fence_after_sync();
#pragma unroll
      for (int c = 0; c < CPT / 32; ++c) tc::tmem_ld32(tl + sb * 128 + c0 + c * 32, s + c * 32);
      tc::tmem_wait_ld();
      tc::fence_before_sync();
      tc::bar_arrive(&s_empty[sb]);
      // raw scores: the max commutes with the positive scale, which is folded
      // into the exponent's FMA below; only the diagonal tile is masked
      if (j == qt) {
        const int lim = r - c0;  // causal: key j*128+c0+c <= row
#pragma unroll
        for (int c = 0; c < CPT; ++c) s[c] = (c <= lim) ? s[c] : -INFINITY;
      }
      float mt = -INFINITY;
#pragma unroll
      for (int c = 0; c < CPT; c += 2) mt = fmaxf(mt, fmaxf(s[c], s[c + 1]));
      mt *= scale_log2;
      if constexpr (NWG > 1) {  // row max over both halves; also orders every S load before any P store
        float* rd = red + (j & 1) * 256;
        rd[wg * 128 + r] = mt;
        prefill_named_bar(1, NSM);
        mt = fmaxf(mt, rd[(1 - wg) * 128 + r]);
      }
      // lazy rescale: move the reference max only when the tile exceeds it by > 2^8
      float corr = 1.f;
      bool resc = false;
      if (mt > m_run + 8.f) {
        corr = (m_run == -INFINITY) ? 0.f : exp2f(m_run - mt);
        resc = j > 0;
        m_run = mt;
        l_run *= corr;
      }
      float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
      for (int c = 0; c < CPT; c += 2) {
        s[c] = ex2_approx(fmaf(s[c], scale_log2, -m_run));
        s[c + 1] = ex2_approx(fmaf(s[c + 1], scale_log2, -m_run));
        ls0 += s[c];
        ls1 += s[c + 1];
      }
      l_run += ls0 + ls1;
      if (__any_sync(0xffffffffu, resc)) {  // O must hold PV(j-1) before it is rescaled
        tc::bar_wait(o_full, (j - 1) & 1u);
        tc::fence_after_sync();
        const float f = resc ? corr : 1.f;
#pragma unroll 1
        for (int c = 0; c < CPT / 32; ++c) {
          float o[32];
          tc::tmem_ld32(tl + 256 + c0 + c * 32, o);
          tc::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= f;
          tc::tmem_st32(tl + 256 + c0 + c * 32, o);
        }
      }
      // P(j) -> TMEM over S(j): hi = p truncated to bf16, lo = (p - hi)
      // truncated; tokens c0+2i, c0+2i+1 -> column (c0/2 + i), low half even.
      // Buffer j&1 was last read by PV(j-2), which completed before S(j) was
      // written (in-order tensor pipe).
#pragma unroll
      for (int c = 0; c < CPT / 32; ++c) {
        const uint32_t col = sb * 128 + c0 / 2 + c * 16;
        if constexpr (PF16) {  // one fp16 P (2^-11 relative) against the fp16 copy of V
          uint32_t ph[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const __half2 h2 = __floats2half2_rn(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]);
            ph[i] = *reinterpret_cast<const uint32_t*>(&h2);
          }
          tc::tmem_st16(tl + col, ph);
        } else {
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float a = s[c * 32 + 2 * i], b = s[c * 32 + 2 * i + 1];
            const uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
            const float ra = a - __uint_as_float(ua & 0xFFFF0000u), rb = b - __uint_as_float(ub & 0xFFFF0000u);
            hi[i] = __byte_perm(ua, ub, 0x7632);
            lo[i] = __byte_perm(__float_as_uint(ra), __float_as_uint(rb), 0x7632);
          }
          tc::tmem_st16(tl + col, hi);
          tc::tmem_st16(tl + col + 64, lo);
        }
      }
      tc::tmem_wait_st();
      tc::fence_before_sync();
      tc::bar_arrive(p_full);
    }
    if constexpr (NWG > 1) {  // row sum over both halves (same m_run in both)
      float* rd = red + (nt & 1) * 256;
      rd[wg * 128 + r] = l_run;
      prefill_named_bar(1, NSM);
      l_run += rd[(1 - wg) * 128 + r];
    }
    tc::bar_wait(o_full, (nt - 1) & 1u);
    tc::fence_after_sync();
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
    const long long obase = (static_cast<long long>(row) * Hq + hq) * 128 + c0;
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(out) + obase;
    float* dstf = static_cast<float*>(out) + obase;
#pragma unroll 1
    for (int c = 0; c < CPT / 32; ++c) {
      float o[32];
      tc::tmem_ld32(tl + 256 + c0 + c * 32, o);
      tc::tmem_wait_ld();
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
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_free<512>(tmem);
}

}  // namespace lkv
