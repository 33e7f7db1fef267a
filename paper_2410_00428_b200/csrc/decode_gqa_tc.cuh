// GQA paged decode attention on the 5th-gen tensor cores (sm_100a tcgen05).
//
// For a GQA group of G query heads sharing one KV head, the decode step is
// two dense contractions per 128-token tile:
//     S^T[128 tok x G] = K[128 tok x 128 d] . Q^T[128 d x G]
//     O^T[128 d  x G] += V^T[128 d x 128 tok] . P^T[128 tok x G]
// On CUDA cores that is 4 FMAs per KV byte at G=8, more than the SM can
// issue at HBM speed (33% of peak). Here both run as
// tcgen05.mma M=128 N=16 K=16 (G padded to 16 with zero rows of Q), so the
// kernel stays HBM-bound. P is split into bf16 hi + lo halves that fill the
// padded columns, so the PV product is accurate to ~2^-16 relative.
//
// Roles, one persistent CTA per SM (224 threads):
//   warp 0   K producer: per unit writes Q into smem (K-major, no swizzle),
//            per tile issues (128/bs) x 2 TMA tensor boxes {64 d, bs tok} of
//            K from the paged slots straight into a swizzle-128B tile (the
//            tensor map spans pool + arena frames, so resident and prefetched
//            blocks are addressed alike through the snapshot);
//   warp 6   V producer: the same for V, on its own ring. A K slot frees when
//            its QK^T completes, a V slot when its PV does, so the softmax is
//            on neither ring's refill cycle;
//   warp 1   MMA issuer (one thread) + TMEM owner: S^T(j) is issued as soon
//            as K(j) lands, PV(j-1) as soon as P(j-1) and V(j-1) are ready;
//   warps 2-5 softmax/epilogue: thread = TMEM lane = token row of S^T and
//            d row of O^T. Lazy running max (a bar.red.or vote; the exact
//            per-head max only when a score exceeds it by 2^8); P^T goes to
//            smem (MN-major, no swizzle) as the B operand of the PV MMA; each
//            tile's O^T lands in a fresh TMEM buffer and is folded into
//            registers with the online-softmax correction (no TMEM
//            read-modify-write hazard).
// Work unit = (chunk of blocks of one sequence, one KV head), exactly as the
// CUDA-core kernel (decode_attn.cuh), and the partial (m, l, o) per query head
// is merged by decode_merge_v3_kernel.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "decode_attn.cuh"
#include "tc_sm100.cuh"

namespace lkv {

template <int G, int BS, int NS>
struct GqaTc {
  static constexpr int kTB = 128 / BS;                 // blocks per 128-token tile
  static constexpr int kTile = 32768;                  // K (or V) tile: 2 SW128 halves of 16 KiB
  static constexpr int kStage = 2 * kTile;             // K + V
  static constexpr int kOffQ = NS * kStage;            // 2 x 4 KiB (Q, K-major none, 16 rows)
  static constexpr int kOffP = kOffQ + 2 * 4096;       // 2 x 4 KiB (P^T, MN-major none)
  static constexpr int kOffRed = kOffP + 2 * 4096;     // [2][4][8] f32 tile maxima
  static constexpr int kOffLred = kOffRed + 256;       // [4][8] f32 row sums
  static constexpr int kOffBar = kOffLred + 128;       // mbarriers
  static constexpr int kNumBars = 4 * NS + 14;
  static constexpr int kOffTmem = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffTmem + 16 + 1024;  // + alignment slack
  static constexpr int kThreads = 224;
  static_assert(kSmem <= 227 * 1024, "smem budget");
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Named barrier that also ORs a predicate over its n threads.
__device__ __forceinline__ bool named_bar_or(int id, int n, bool v) {
  uint32_t r;
  asm volatile(
      "{\n"
      ".reg .pred p, q;\n"
      "setp.ne.u32 p, %1, 0;\n"
      "bar.red.or.pred q, %2, %3, p;\n"
      "selp.u32 %0, 1, 0, q;\n"
      "}\n"
      : "=r"(r)
      : "r"(static_cast<uint32_t>(v)), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}

// Lazy running max (log2 domain): a tile rescales only when one of its scores
// exceeds the running max of its head by more than this (exp2 <= 2^8 keeps P
// and the fp32 sums far from overflow), so most tiles skip the max reduction.
constexpr float kLazyMax = 8.f;

template <int G, int BS, int NS>
__global__ void __launch_bounds__(224, 1) decode_gqa_tc_kernel(
    const __grid_constant__ CUtensorMap kvmap, int Hl, const int* __restrict__ snap,
    const AttnSeq* __restrict__ seqs, const AttnChunk* __restrict__ chunks, int n_units,
    const __nv_bfloat16* __restrict__ q, float* __restrict__ part_o, float* __restrict__ part_ml,
    float scale_log2, unsigned long long* stamps) {
  using C = GqaTc<G, BS, NS>;
  constexpr int TB = C::kTB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::kOffBar);
  uint64_t* kfull = bars;            // [NS] K half landed (TMA -> MMA)
  uint64_t* kempty = bars + NS;      // [NS] QK^T done with the K half
  uint64_t* vfull = bars + 2 * NS;   // [NS] V half landed
  uint64_t* vempty = bars + 3 * NS;  // [NS] PV done with the V half
  uint64_t* s_full = bars + 4 * NS;  // [2] S^T in TMEM
  uint64_t* s_empty = s_full + 2;    // [2] S^T read by softmax
  uint64_t* p_full = s_full + 4;     // [2] P^T in smem
  uint64_t* o_full = s_full + 6;     // [2] O^T tile in TMEM
  uint64_t* o_empty = s_full + 8;    // [2] O^T tile read
  uint64_t* q_full = s_full + 10;    // [2] Q in smem
  uint64_t* q_empty = s_full + 12;   // [2] last QK^T of the unit done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + C::kOffTmem);
  float* red = reinterpret_cast<float*>(sm + C::kOffRed);
  float* lred = reinterpret_cast<float*>(sm + C::kOffLred);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      tc::bar_init(&kfull[s], 1);
      tc::bar_init(&kempty[s], 1);
      tc::bar_init(&vfull[s], 1);
      tc::bar_init(&vempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::bar_init(&s_full[b], 1);
      tc::bar_init(&s_empty[b], 128);
      tc::bar_init(&p_full[b], 128);
      tc::bar_init(&o_full[b], 1);
      tc::bar_init(&o_empty[b], 128);
      tc::bar_init(&q_full[b], 1);
      tc::bar_init(&q_empty[b], 1);
    }
    tc::bar_fence_init();
  }
  // Q and P^T buffers: rows/columns beyond G stay zero for the whole kernel.
  for (int i = threadIdx.x; i < 4 * 4096 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm + C::kOffQ)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 1) tc::tmem_alloc<64>(tmem_slot);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  const int rows_per_frame = 2 * Hl * BS;
  pdl_launch_dependents();
  stamp_begin(stamps);

  if (warp == 0 || warp == 6) {
    // ------------------------------------------------------------ producers
    // warp 0 loads Q and the K half of each tile, warp 6 the V half. The two
    // halves have their own rings: a K slot frees as soon as its QK^T is done,
    // a V slot when its PV is, so the softmax sits on neither ring's cycle.
    const bool kside = warp == 0;
    uint64_t* ring_full = kside ? kfull : vfull;
    uint64_t* ring_empty = kside ? kempty : vempty;
    int stage = 0, qb = 0;
    uint32_t ph = 0, qph = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const AttnChunk ck = chunks[u / Hl];
      const int h = u % Hl;
      const AttnSeq sd = seqs[ck.seq];
      if (kside) {
        tc::bar_wait(&q_empty[qb], qph ^ 1u);
        // Q rows g < G: chunk c = (g, d8) -> (d8 * 128 + g * 16) in the K-major core-matrix layout
        const __nv_bfloat16* qs = q + (static_cast<long long>(ck.seq) * Hl + h) * G * 128;
        uint8_t* qd = sm + C::kOffQ + qb * 4096;
        for (int c = lane; c < G * 16; c += 32) {
          const int g = c >> 4, d8 = c & 15;
          *reinterpret_cast<uint4*>(qd + d8 * 128 + g * 16) =
              *reinterpret_cast<const uint4*>(qs + g * 128 + d8 * 8);
        }
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) tc::bar_arrive(&q_full[qb]);
        if (++qb == 2) {
          qb = 0;
          qph ^= 1u;
        }
      }
      const int ntile = (ck.nb + TB - 1) / TB;
      for (int t = 0; t < ntile; ++t) {
        int frame = 0;
        if (lane < TB) {
          const int bi = min(t * TB + lane, ck.nb - 1);
          frame = snap[sd.blk_offset + ck.b0 + bi];
        }
        if (lane == 0) {
          tc::bar_wait(&ring_empty[stage], ph ^ 1u);
          tc::bar_expect_tx(&ring_full[stage], C::kTile);
        }
        __syncwarp();
        if (lane < TB) {
          const int rk = frame * rows_per_frame + h * BS;
          const int row = kside ? rk : rk + Hl * BS;
          uint8_t* dst = sm + stage * C::kStage + (kside ? 0 : C::kTile) + lane * BS * 128;
#pragma unroll
          for (int half = 0; half < 2; ++half) tc::tma_load_2d(dst + half * 16384, &kvmap, half * 64, row, &ring_full[stage]);
        }
        __syncwarp();
        if (++stage == NS) {
          stage = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = tc::idesc_bf16(128, 16, false, false);
      constexpr uint32_t idO = tc::idesc_bf16(128, 16, true, true);
      const uint32_t kv0 = tc::saddr(sm), q0 = tc::saddr(sm + C::kOffQ), p0 = tc::saddr(sm + C::kOffP);
      int stage = 0, qb = 0;
      uint32_t ph = 0, qph = 0;
      unsigned j = 0;
      bool have_prev = false;
      int prev_stage = 0;
      uint32_t prev_ph = 0;
      unsigned prev_j = 0;
      auto pv_ready = [&]() {
        return tc::bar_test(&p_full[prev_j & 1], (prev_j >> 1) & 1u) && tc::bar_test(&vfull[prev_stage], prev_ph);
      };
      auto issue_pv = [&]() {
        const int pb = prev_j & 1;
        const uint32_t par = (prev_j >> 1) & 1u;
        tc::bar_wait(&p_full[pb], par);
        tc::bar_wait(&o_empty[pb], par ^ 1u);
        tc::bar_wait(&vfull[prev_stage], prev_ph);
        tc::fence_after_sync();
        const uint32_t vt = kv0 + prev_stage * C::kStage + C::kTile;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::mma_bf16(tmem + 32 + pb * 16, tc::smem_desc(vt + kk * 2048, 16384, 1024, tc::kLayoutSw128),
                       tc::smem_desc(p0 + pb * 4096 + kk * 512, 256, 128, tc::kLayoutNone), idO, kk > 0);
        tc::mma_commit(&o_full[pb]);
        tc::mma_commit(&vempty[prev_stage]);
        have_prev = false;
      };
      // PV(j-1) frees a V slot: issue it as soon as P(j-1) and V(j-1) are
      // there, while waiting for whatever the next QK^T needs.
      auto wait_or_pv = [&](uint64_t* bar, uint32_t parity) {
        if (!have_prev) return;
        while (!tc::bar_test(bar, parity)) {
          if (pv_ready()) {
            issue_pv();
            return;
          }
        }
      };
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const AttnChunk ck = chunks[u / Hl];
        const int ntile = (ck.nb + TB - 1) / TB;
        wait_or_pv(&q_full[qb], qph);
        tc::bar_wait(&q_full[qb], qph);
        for (int t = 0; t < ntile; ++t) {
          const int sb = j & 1;
          wait_or_pv(&kfull[stage], ph);
          tc::bar_wait(&kfull[stage], ph);
          tc::bar_wait(&s_empty[sb], ((j >> 1) & 1u) ^ 1u);
          tc::fence_after_sync();
          const uint32_t kt = kv0 + stage * C::kStage;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            tc::mma_bf16(tmem + sb * 16,
                         tc::smem_desc(kt + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, tc::kLayoutSw128),
                         tc::smem_desc(q0 + qb * 4096 + kk * 256, 128, 2048, tc::kLayoutNone), idS, kk > 0);
          tc::mma_commit(&s_full[sb]);
          tc::mma_commit(&kempty[stage]);
          if (t == ntile - 1) tc::mma_commit(&q_empty[qb]);
          if (have_prev) issue_pv();
          have_prev = true;
          prev_stage = stage;
          prev_ph = ph;
          prev_j = j;
          ++j;
          if (++stage == NS) {
            stage = 0;
            ph ^= 1u;
          }
        }
        if (++qb == 2) {
          qb = 0;
          qph ^= 1u;
        }
      }
      if (have_prev) issue_pv();
    }
  } else if (warp <= 5) {
    // ------------------------------------------------------------ softmax / epilogue
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // TMEM lane: token row of S^T, d row of O^T
    const uint32_t tl = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    unsigned j = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const AttnChunk ck = chunks[u / Hl];
      const int kv_len = seqs[ck.seq].kv_len;
      const int ntile = (ck.nb + TB - 1) / TB;
      float m_run[G], l_part[G], o_acc[G], corr_prev[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        m_run[g] = -INFINITY;
        l_part[g] = 0.f;
        o_acc[g] = 0.f;
        corr_prev[g] = 0.f;
      }
      auto epilogue = [&](unsigned jj) {
        const int ob = jj & 1;
        tc::bar_wait(&o_full[ob], (jj >> 1) & 1u);
        tc::fence_after_sync();
        float o[16];
        tc::tmem_ld16(tl + 32 + ob * 16, o);
        tc::tmem_wait_ld();
        tc::reg_fence<16>(o);
        tc::fence_before_sync();
        tc::bar_arrive(&o_empty[ob]);
#pragma unroll
        for (int g = 0; g < G; ++g) o_acc[g] = fmaf(o_acc[g], corr_prev[g], o[g] + o[8 + g]);
      };
      for (int t = 0; t < ntile; ++t) {
        const int sb = j & 1;
        tc::bar_wait(&s_full[sb], (j >> 1) & 1u);
        tc::fence_after_sync();
        float s[8];
        tc::tmem_ld8(tl + sb * 16, s);
        tc::tmem_wait_ld();
        tc::reg_fence<8>(s);
        tc::fence_before_sync();
        tc::bar_arrive(&s_empty[sb]);
        const int bi = t * TB + r / BS;
        const int tok = (ck.b0 + bi) * BS + (r % BS);
        const bool valid = bi < ck.nb && tok < kv_len;
        bool raise = false;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          s[g] = valid ? s[g] * scale_log2 : -INFINITY;
          raise |= s[g] > m_run[g] + kLazyMax;  // -inf running max: any valid score raises
        }
        float corr[G];
        float p[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) p[g] = 0.f;
        if (named_bar_or(1, 128, raise)) {  // uniform: some head's max moved too far, reduce exactly
          float* rd = red + (j & 1) * 32;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            float mx = s[g];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if (lane == 0) rd[quad * 8 + g] = mx;
          }
          named_bar_sync(1, 128);
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float tmax = fmaxf(fmaxf(rd[g], rd[8 + g]), fmaxf(rd[16 + g], rd[24 + g]));
            const float mnew = fmaxf(m_run[g], tmax);
            corr[g] = (m_run[g] == -INFINITY) ? 0.f : exp2f(m_run[g] - mnew);
            m_run[g] = mnew;
          }
        } else {
#pragma unroll
          for (int g = 0; g < G; ++g) corr[g] = 1.f;
        }
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          p[g] = (s[g] == -INFINITY) ? 0.f : exp2f(s[g] - m_run[g]);
          l_part[g] = fmaf(l_part[g], corr[g], p[g]);
        }
        // P = hi + lo, both bf16 (columns g and 8+g of the N=16 operand): the
        // PV product keeps ~16 mantissa bits of P at no extra MMA cost, which
        // holds the 1e-3 relative bar even for a handful of tokens.
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          hi[i] = tc::pack_bf16(p[2 * i], p[2 * i + 1]);
          const float h0 = __uint_as_float(hi[i] << 16), h1 = __uint_as_float(hi[i] & 0xFFFF0000u);
          lo[i] = tc::pack_bf16(p[2 * i] - h0, p[2 * i + 1] - h1);
        }
        // P^T row r (MN-major core matrices: (r/8)*256 + n*128 + (r%8)*16); buffer
        // j&1 was last read by PV(j-2), whose completion this thread already observed.
        uint8_t* prow = sm + C::kOffP + (j & 1) * 4096 + (r >> 3) * 256 + (r & 7) * 16;
        *reinterpret_cast<uint4*>(prow) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(prow + 128) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        tc::fence_async_smem();
        tc::bar_arrive(&p_full[j & 1]);
        if (t > 0) epilogue(j - 1);
#pragma unroll
        for (int g = 0; g < G; ++g) corr_prev[g] = corr[g];
        ++j;
      }
      epilogue(j - 1);
      // unit epilogue: sum the per-token partial row sums, write (m, l, o)
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float l = l_part[g];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        if (lane == 0) lred[quad * 8 + g] = l;
      }
      named_bar_sync(1, 128);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const long long pu = static_cast<long long>(u) * G + g;
        part_o[pu * 128 + r] = o_acc[g];
        if (r == 0) {
          part_ml[pu * 2 + 0] = m_run[g];
          part_ml[pu * 2 + 1] = lred[g] + lred[8 + g] + lred[16 + g] + lred[24 + g];
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_free<64>(tmem);
  if (warp == 0) stamp_end(stamps);
}

}  // namespace lkv
