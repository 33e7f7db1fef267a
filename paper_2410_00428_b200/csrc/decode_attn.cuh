// Paged decode attention for sm_100a: persistent warps fed by TMA bulk copies.
//
// The kernel is HBM-bound (every K/V byte is read once, ~1-8 FMAs per byte),
// so the design goal is keeping enough bytes in flight per SM, not math.
//
//  * Work unit = (chunk of <= 32 blocks of one sequence, one KV head). Units
//    are dealt round-robin to every warp of a persistent grid (one CTA per SM),
//    so ragged batches and long contexts load-balance without a tail wave.
//  * Each warp streams its units' 16-token sub-tiles (4 KiB K + 4 KiB V per
//    head, contiguous in the slot layout) through a private S-stage shared-
//    memory ring filled by cp.async.bulk (TMA bulk copy engine, SASS UBLKCP)
//    and tracked by one mbarrier per stage (expect_tx / complete_tx). Lane 0
//    refills a stage as soon as the warp has consumed it, so S-1 sub-tiles are
//    always in flight per warp. No registers are spent on staging.
//  * The block table is staged per unit: lane j holds block j's frame.
//  * Math per sub-tile: lane (c = dims 8c..8c+7, r0 = row parity) reads rows
//    r0 + 2k with conflict-free 16 B shared loads; Q.K partials are reduced by
//    a value-splitting butterfly (8 shuffles for 8 rows); online softmax in
//    the log2 domain; P.V in fp32. G query heads of a GQA group share every
//    K/V byte.
//  * Each unit writes an unnormalised partial (m, l, o), merged per
//    (sequence, query head) by decode_merge_v5_kernel (one CTA each).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lkv {

struct AttnChunk {
  int seq;   // batch member
  int b0;    // first block
  int nb;    // blocks in the chunk (<= 32)
  int pad;
};

struct AttnSeq {
  int blk_offset;  // member's first snapshot entry
  int kv_len;
  int chunk0;      // first chunk of the member
  int nchunk;
};

// Programmatic dependent launch: the attention kernels let the split merge
// launch early (its CTAs are dispatched next to the persistent attention CTAs
// and park in griddepcontrol.wait until the attention grid has completed and
// flushed), so the merge's launch latency hides under the attention kernel.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Kernel span stamps (timing mode): the first CTA's start and the last
// warp's end on %globaltimer, so the attention kernel's own duration can be
// told apart from launch latency in the event-timed interval.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// st[0] keeps ~start (atomicMax of the complement = earliest start), so a
// zeroed pair is the initial state.
__device__ __forceinline__ void stamp_begin(unsigned long long* st) {
  if (st && threadIdx.x == 0) atomicMax(st, ~global_ns());
}
__device__ __forceinline__ void stamp_end(unsigned long long* st) {
  if (st && (threadIdx.x & 31) == 0) atomicMax(st + 1, global_ns());
}

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LKV_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LKV_WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ uint4 lds128(const char* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_addr(p)));
  return r;
}

__device__ __forceinline__ void cvt8(const uint4& u, float* f) {
  f[0] = __uint_as_float(u.x << 16);
  f[1] = __uint_as_float(u.x & 0xFFFF0000u);
  f[2] = __uint_as_float(u.y << 16);
  f[3] = __uint_as_float(u.y & 0xFFFF0000u);
  f[4] = __uint_as_float(u.z << 16);
  f[5] = __uint_as_float(u.z & 0xFFFF0000u);
  f[6] = __uint_as_float(u.w << 16);
  f[7] = __uint_as_float(u.w & 0xFFFF0000u);
}

constexpr int kSubTok = 16;                   // tokens per sub-tile
constexpr int kHeadDim = 128;
constexpr int kSubBytes = kSubTok * kHeadDim * 2;  // 4 KiB of K (or V) per head

template <int G, int BS, int W, int S>
struct AttnV2 {
  static constexpr int kThreads = W * 32;
  static constexpr int kStageBytes = 2 * kSubBytes;
  static constexpr int kSmem = W * S * kStageBytes + W * S * 8;
  static constexpr int kSubPerBlock = BS / kSubTok;
};

template <int G, int BS, int W, int S>
__global__ void __launch_bounds__(W * 32, 1) decode_attn_v2_kernel(
    const char* __restrict__ base, long long slot_bytes, int Hl, const int* __restrict__ snap,
    const AttnSeq* __restrict__ seqs, const AttnChunk* __restrict__ chunks, int n_units,
    const __nv_bfloat16* __restrict__ q, float* __restrict__ part_o, float* __restrict__ part_ml,
    float scale_log2, unsigned long long* stamps) {
  using C = AttnV2<G, BS, W, S>;
  constexpr int D = kHeadDim;
  constexpr int SUB = C::kSubPerBlock;
  extern __shared__ __align__(128) char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = lane & 15, r0 = lane >> 4;
  char* ring = smem + warp * S * C::kStageBytes;
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(smem + W * S * C::kStageBytes) + warp * S;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  pdl_launch_dependents();
  stamp_begin(stamps);
  const int gw = blockIdx.x * W + warp;
  const int NW = gridDim.x * W;
  const long long tile_bytes = static_cast<long long>(BS) * D * 2;
  const long long v_off = static_cast<long long>(Hl) * tile_bytes;

  // ---- issue side: walks the same unit/sub-tile sequence as the compute side
  int iu = gw, it = 0, i_nsub = 0, i_h = 0, i_frame = 0;
  auto issue_unit_info = [&]() {
    if (iu >= n_units) return;
    const AttnChunk ck = chunks[iu / Hl];
    i_h = iu % Hl;
    i_nsub = ck.nb * SUB;
    const int off = seqs[ck.seq].blk_offset + ck.b0;
    i_frame = lane < ck.nb ? snap[off + lane] : 0;
  };
  int issued = 0;
  auto issue_next = [&]() {
    if (iu >= n_units) return;
    const int frame = __shfl_sync(0xffffffffu, i_frame, it / SUB);
    if (lane == 0) {
      const int st = issued % S;
      char* dst = ring + st * C::kStageBytes;
      const char* kp = base + static_cast<long long>(frame) * slot_bytes + i_h * tile_bytes +
                       (it % SUB) * kSubBytes;
      mbar_expect_tx(&bars[st], C::kStageBytes);
      bulk_g2s(dst, kp, kSubBytes, &bars[st]);
      bulk_g2s(dst + kSubBytes, kp + v_off, kSubBytes, &bars[st]);
    }
    ++issued;
    if (++it == i_nsub) {
      it = 0;
      iu += NW;
      issue_unit_info();
    }
  };
  issue_unit_info();
  for (int s = 0; s < S; ++s) issue_next();

  // ---- compute side
  int consumed = 0;
  unsigned phases = 0;
  for (int u = gw; u < n_units; u += NW) {
    const AttnChunk ck = chunks[u / Hl];
    const int h = u % Hl;
    const int kv_len = seqs[ck.seq].kv_len;
    const int nsub = ck.nb * SUB;
    float qf[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint4 qu = *reinterpret_cast<const uint4*>(
          q + (static_cast<long long>(ck.seq) * Hl * G + h * G + g) * D + c * 8);
      cvt8(qu, qf[g]);
#pragma unroll
      for (int i = 0; i < 8; ++i) qf[g][i] *= scale_log2;
    }
    float mrun[G], lrun[G], acc[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      mrun[g] = -INFINITY;
      lrun[g] = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[g][i] = 0.f;
    }
    for (int t = 0; t < nsub; ++t) {
      const int st = consumed % S;
      mbar_wait(&bars[st], (phases >> st) & 1u);
      phases ^= 1u << st;
      const char* kt = ring + st * C::kStageBytes + (r0 * D + c * 8) * 2;
      const char* vt = kt + kSubBytes;
      const int tok0 = (ck.b0 + t / SUB) * BS + (t % SUB) * kSubTok;
      const bool full_tile = tok0 + kSubTok <= kv_len;
      uint4 kr[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) kr[k] = lds128(kt + k * 2 * D * 2);
      float s[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float pr[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float kf[8];
          cvt8(kr[k], kf);
          float a = 0.f;
#pragma unroll
          for (int i = 0; i < 8; ++i) a = fmaf(qf[g][i], kf[i], a);
          pr[k] = a;
        }
        const bool b3 = c & 8, b2 = c & 4, b1 = c & 2;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float send = b3 ? pr[j] : pr[j + 4];
          const float keep = b3 ? pr[j + 4] : pr[j];
          pr[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const float send = b2 ? pr[j] : pr[j + 2];
          const float keep = b2 ? pr[j + 2] : pr[j];
          pr[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        {
          const float send = b1 ? pr[0] : pr[1];
          const float keep = b1 ? pr[1] : pr[0];
          pr[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
        pr[0] += __shfl_xor_sync(0xffffffffu, pr[0], 1);
        s[g] = (full_tile || tok0 + r0 + (c & 14) < kv_len) ? pr[0] : -INFINITY;
      }
      uint4 vr[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) vr[k] = lds128(vt + k * 2 * D * 2);
      // stage fully read: hand it back to the copy engine
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      ++consumed;
      issue_next();
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float mt = s[g];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, o));
        const float mnew = fmaxf(mrun[g], mt);
        const float corr = (mrun[g] == -INFINITY) ? 0.f : exp2f(mrun[g] - mnew);
        const float p = (s[g] == -INFINITY) ? 0.f : exp2f(s[g] - mnew);
        lrun[g] = lrun[g] * corr + ((c & 1) ? 0.f : p);
        mrun[g] = mnew;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[g][i] *= corr;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float pk = __shfl_sync(0xffffffffu, p, (lane & 16) + 2 * k);
          float vf[8];
          cvt8(vr[k], vf);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[g][i] = fmaf(pk, vf[i], acc[g][i]);
        }
      }
    }
    // ---- unit epilogue: unnormalised partial (m, l, o) per query head
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[g][i] += __shfl_xor_sync(0xffffffffu, acc[g][i], 16);
      float l = lrun[g];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
      const long long pu = static_cast<long long>(u) * G + g;
      if (lane < 16) {
        float4* dst = reinterpret_cast<float4*>(part_o + pu * D + c * 8);
        dst[0] = make_float4(acc[g][0], acc[g][1], acc[g][2], acc[g][3]);
        dst[1] = make_float4(acc[g][4], acc[g][5], acc[g][6], acc[g][7]);
      }
      if (lane == 0) {
        part_ml[pu * 2 + 0] = mrun[g];
        part_ml[pu * 2 + 1] = l;
      }
    }
  }
  stamp_end(stamps);
}

// Fused all-gather of the per-head outputs (the path's one
// exchange). Every rank's gather buffer (cudaMalloc'd by its lkv_device,
// opened by the peers through CUDA IPC) is
//   [flags: kGatherFlagWords u32][rows: 2 parities x max_batch x Hq_total x 128 bf16]
// The merge writes each final row into every rank's buffer at this rank's
// head offset; the last CTA of the launch then raises flags[tp_rank] = epoch
// in every buffer (release at system scope). A consumer waits for all flags.
constexpr int kGatherFlagWords = 64;
struct GatherArgs {
  char* const* bases;   // device array [n] of gather buffer bases (peer pointers), or nullptr
  int n;                // ranks
  int rank;             // this rank = index of its own flag word
  int hq_total;         // query heads over all ranks
  int max_batch;
  int parity;           // epoch & 1: row buffer of this layer
  unsigned epoch;
  unsigned* done;       // CTA completion counter (self re-arming)
};

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// A layer with no members still publishes its epoch.
__global__ void gather_flag_kernel(GatherArgs ga) {
  __threadfence_system();
  for (int p = 0; p < ga.n; ++p) st_release_sys(reinterpret_cast<unsigned*>(ga.bases[p]) + ga.rank, ga.epoch);
}

// Waits until every rank raised its flag to `epoch` in this rank's buffer.
__global__ void gather_wait_kernel(const unsigned* __restrict__ flags, int n, unsigned epoch) {
  const int i = threadIdx.x;
  if (i < n) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (static_cast<int>(ld_acquire_sys(flags + i) - epoch) < 0) {
      __nanosleep(256);
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) __trap();  // a rank never published: fail loudly, do not hang
    }
  }
  __syncwarp();
}

// Writes merged row (member m, query head hq): lane owns dims 4*lane..+3.
// Also stores the row into every rank's gather buffer and, from the launch's
// last CTA, publishes the epoch (fused all-gather). Called by
// all threads of the CTA; warp 0 holds the row.
__device__ __forceinline__ void merge_store_row(float4 r, float Lt, int m, int hq, int Hl, int G, void* out,
                                                int out_f32, const GatherArgs& ga) {
  if ((threadIdx.x >> 5) == 0) {
    const int lane = threadIdx.x & 31;
    const float inv = Lt > 0.f ? 1.f / Lt : 0.f;
    const long long idx = (static_cast<long long>(m) * Hl * G + hq) * kHeadDim + lane * 4;
    uint2 pk;
    pk.x = (static_cast<unsigned>(__bfloat16_as_ushort(__float2bfloat16_rn(r.y * inv))) << 16) |
           __bfloat16_as_ushort(__float2bfloat16_rn(r.x * inv));
    pk.y = (static_cast<unsigned>(__bfloat16_as_ushort(__float2bfloat16_rn(r.w * inv))) << 16) |
           __bfloat16_as_ushort(__float2bfloat16_rn(r.z * inv));
    if (out_f32)
      *reinterpret_cast<float4*>(static_cast<float*>(out) + idx) = make_float4(r.x * inv, r.y * inv, r.z * inv, r.w * inv);
    else
      *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(out) + idx) = pk;
    if (ga.bases) {  // this row into every rank's gather buffer (NVLink stores to peers)
      const long long row = (static_cast<long long>(ga.parity) * ga.max_batch + m) * ga.hq_total +
                            static_cast<long long>(ga.rank) * Hl * G + hq;
      const long long off = kGatherFlagWords * 4 + row * kHeadDim * 2 + lane * 8;
      for (int p = 0; p < ga.n; ++p) *reinterpret_cast<uint2*>(ga.bases[p] + off) = pk;
    }
  }
  if (ga.bases) {  // the launch's last CTA publishes the epoch to every rank
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned total = gridDim.x * gridDim.y;
      if (atomicAdd(ga.done, 1u) == total - 1) {
        __threadfence_system();
        for (int p = 0; p < ga.n; ++p)
          st_release_sys(reinterpret_cast<unsigned*>(ga.bases[p]) + ga.rank, ga.epoch);
        *ga.done = 0u;
      }
    }
  }
}

// Merge v5: one CTA (W warps) per (member, query head), a single pass. Warp w
// folds chunks w, w+W, ... in batches of 8 with every load of a batch issued
// before any math, and keeps its own running max (rescaling its sum when a
// batch raises it), so no separate max pass costs a memory round trip; the
// W (max, sum, row) partials meet in shared memory. 8W loads of 512 B in
// flight per CTA: the merge is latency-bound (few CTAs, L2-resident partials).
// W=4 (~110 registers x 128 threads) fits beside a persistent attention CTA,
// which is what programmatic dependent launch needs to overlap the two.
template <int W>
__global__ void __launch_bounds__(W * 32) decode_merge_v5_kernel(const float* __restrict__ part_o,
                                                               const float* __restrict__ part_ml,
                                                               const AttnSeq* __restrict__ seqs, int Hl, int G,
                                                               void* __restrict__ out, int out_f32,
                                                               GatherArgs ga) {
  constexpr int B = 8;
  __shared__ float4 so[W][32];
  __shared__ float sm_[W], sl_[W];
  pdl_wait();  // partials of the attention grid (no-op without PDL)
  const int m = blockIdx.x, hq = blockIdx.y, h = hq / G, g = hq % G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const AttnSeq sd = seqs[m];
  const int nch = sd.nchunk;
  const long long cstride = static_cast<long long>(Hl) * G;
  const long long pu0 = (static_cast<long long>(sd.chunk0) * Hl + h) * G + g;
  float M = -INFINITY, L = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c0 = warp; c0 < nch; c0 += W * B) {
    float4 v[B];
    float2 ml[B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const int c = c0 + W * i;
      if (c < nch) {
        const long long pu = pu0 + c * cstride;
        v[i] = __ldcg(reinterpret_cast<const float4*>(part_o + pu * kHeadDim) + lane);
        ml[i] = __ldcg(reinterpret_cast<const float2*>(part_ml + pu * 2));
      } else {
        v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        ml[i] = make_float2(-INFINITY, 0.f);
      }
    }
    float mb = M;
#pragma unroll
    for (int i = 0; i < B; ++i) mb = fmaxf(mb, ml[i].x);
    if (mb == -INFINITY) continue;  // nothing valid yet
    const float cs = (M == -INFINITY) ? 0.f : exp2f(M - mb);
    L *= cs;
    acc.x *= cs;
    acc.y *= cs;
    acc.z *= cs;
    acc.w *= cs;
    M = mb;
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const float f = (ml[i].x == -INFINITY) ? 0.f : exp2f(ml[i].x - M);
      L = fmaf(f, ml[i].y, L);
      acc.x = fmaf(f, v[i].x, acc.x);
      acc.y = fmaf(f, v[i].y, acc.y);
      acc.z = fmaf(f, v[i].z, acc.z);
      acc.w = fmaf(f, v[i].w, acc.w);
    }
  }
  so[warp][lane] = acc;
  if (lane == 0) {
    sm_[warp] = M;
    sl_[warp] = L;
  }
  __syncthreads();
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  float Lt = 0.f;
  if (warp == 0) {
    float Mg = -INFINITY;
#pragma unroll
    for (int w = 0; w < W; ++w) Mg = fmaxf(Mg, sm_[w]);
    if (Mg != -INFINITY) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const float f = (sm_[w] == -INFINITY) ? 0.f : exp2f(sm_[w] - Mg);
        const float4 a = so[w][lane];
        Lt = fmaf(f, sl_[w], Lt);
        r.x = fmaf(f, a.x, r.x);
        r.y = fmaf(f, a.y, r.y);
        r.z = fmaf(f, a.z, r.z);
        r.w = fmaf(f, a.w, r.w);
      }
    }
  }
  merge_store_row(r, Lt, m, hq, Hl, G, out, out_f32, ga);
}

}  // namespace lkv
