// sm_100a kernels of the LayerKV data path. All of them are HBM-bound byte
// movers or (decode attention) HBM-bound streaming reductions; none is
// GEMM-shaped, so none uses tensor cores.
//
// Slot layout (one (block, layer) slot of one GPU's KV-head shard):
//   [K | V][kv_heads_local][tokens_per_block][head_dim]  bf16
// so one (slot, head) K or V tile is tokens_per_block * head_dim * 2 bytes
// contiguous (4 KiB at bs=16, d=128).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kvgen.cuh"

namespace lkv {

struct uint4_ {
  unsigned x, y, z, w;
};

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// ---------------------------------------------------------------------------
// Block-table mirror: apply a journal of (index, value) updates. The journal
// lives in pinned host memory and is read over the link directly (8-16 B per
// update; a 32k-token allocation is 65 k updates).
struct TableUpdate {
  long long index;
  int value;
  int pad;
};

// Device mirror of the two LIFO free lists (reference SlotPool,
// kv_manager.cpp:52-74). A stack is [total-1 ... next_fresh] + pushed[0..size)
// (kv_manager.hpp FreeListDelta); a sync writes the changed tail
// pushed[low..size) and the header {total, next_fresh, size}. List 0 = GPU,
// 1 = CPU.
struct FreeSync {
  const unsigned* src[2];  // uploaded pushed[low..size) of each list
  unsigned* dst[2];        // device stacks
  long long low[2], n[2], total[2], fresh[2], size[2];
  long long* hdr;          // [2][3] = {total, next_fresh, pushed size} per list
  int any;
};

// Applies a batch of block-table updates (last update per entry only, see
// lkv_device::dedupe_journal) and, in the same launch, the free-list sync.
__global__ void table_apply_kernel(const TableUpdate* __restrict__ upd, int n,
                                   int* __restrict__ table, FreeSync fs) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) {
    const TableUpdate u = upd[i];
    table[u.index] = u.value;
  }
  if (!fs.any) return;
#pragma unroll
  for (int l = 0; l < 2; ++l)
    for (long long i = tid; i < fs.n[l]; i += nt) fs.dst[l][fs.low[l] + i] = fs.src[l][i];
  if (tid == 0)
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      fs.hdr[3 * l] = fs.total[l];
      fs.hdr[3 * l + 1] = fs.fresh[l];
      fs.hdr[3 * l + 2] = fs.size[l];
    }
}

// ---------------------------------------------------------------------------
// Scatter / pack: contiguous prefill output K,V [tokens][Hl][D] -> slots.
// Block b (tokens [b*bs, b*bs+bs)) goes to dst + frame[b] * slot_bytes, where
// frame = the GPU slot ids from the table mirror (retained layer, scatter)
// or b - b0 (offloaded layer, pack into a staging segment; rev_n > 0: rev_n -
// 1 - (b - b0), the span packed in reverse so that descending CPU slots, as
// the LIFO free list hands out a released request's slots, still meet the
// staging in ascending order and their D2H coalesces into one copy). Tokens past
// `tokens` in the tail block are zero-filled.
// One CTA per half slot (K or V of block b0 + i): [Hl][bs][128] bf16, written
// contiguously; source rows (token, head) of the prefill K/V. 32-bit index
// math (bs = 1 << bs_shift, D = 128) and 4 independent 16 B loads in flight
// per thread.
__global__ void __launch_bounds__(256) scatter_slots_kernel(const __nv_bfloat16* __restrict__ k,
                                                            const __nv_bfloat16* __restrict__ v, long long tokens,
                                                            int b0, const int* __restrict__ frames,
                                                            char* __restrict__ dst, long long slot_bytes, int Hl,
                                                            int bs_shift, int rev_n) {
  const int half = static_cast<int>(blockIdx.x & 1u);
  const int bl = static_cast<int>(blockIdx.x >> 1);
  const int b = b0 + bl;
  const long long frame = frames ? frames[b] : (rev_n > 0 ? rev_n - 1 - bl : bl);
  char* out = dst + frame * slot_bytes + half * (slot_bytes >> 1);
  const __nv_bfloat16* src = half ? v : k;
  const int bs_mask = (1 << bs_shift) - 1;
  const int nvec = (Hl << bs_shift) << 4;  // 16 vectors of 8 bf16 per (head, token) row
  const long long tok0 = static_cast<long long>(b) << bs_shift;
  for (int j0 = threadIdx.x; j0 < nvec; j0 += 4 * blockDim.x) {
    uint4 val[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * blockDim.x;
      val[u] = make_uint4(0, 0, 0, 0);
      if (j < nvec) {
        const int c = j & 15, row = j >> 4;
        const long long tok = tok0 + (row & bs_mask);
        if (tok < tokens) val[u] = ld_stream(src + ((tok * Hl + (row >> bs_shift)) << 7) + c * 8);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * blockDim.x;
      if (j < nvec) st_stream(out + static_cast<long long>(j) * 16, val[u]);
    }
  }
}

// One CTA per slot: pool slot slots[i] -> dst + i * slot_bytes (the
// escalation gather into staging), 4 x 16 B loads in flight per thread.
__global__ void __launch_bounds__(256) gather_slots_v2_kernel(const char* __restrict__ pool,
                                                              const unsigned* __restrict__ slots,
                                                              long long slot_bytes, char* __restrict__ dst) {
  const char* src = pool + static_cast<long long>(slots[blockIdx.x]) * slot_bytes;
  char* out = dst + static_cast<long long>(blockIdx.x) * slot_bytes;
  const int nvec = static_cast<int>(slot_bytes >> 4);
  for (int j0 = threadIdx.x; j0 < nvec; j0 += 4 * blockDim.x) {
    uint4 val[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * blockDim.x;
      if (j < nvec) val[u] = ld_stream(src + static_cast<long long>(j) * 16);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * blockDim.x;
      if (j < nvec) st_stream(out + static_cast<long long>(j) * 16, val[u]);
    }
  }
}

// Tiered prefetch (f3): pull pinned host frames over the link into the arena
// with SM loads, one launch per layer instead of one copy-engine transfer per
// scattered frame (the read-in hands out frames in LRU order, so a layer's
// frames rarely form runs). pairs[i] = {host frame, arena frame}; host frames
// are mapped pinned memory. A persistent grid walks the frames; each thread
// keeps 8 x 16 B loads in flight (the link's latency-bandwidth product is
// ~100 KB, so a few dozen CTAs saturate it).
struct FramePair {
  long long src, dst;
};

__global__ void __launch_bounds__(256) pull_frames_kernel(const char* __restrict__ host, char* __restrict__ dev,
                                                          const FramePair* __restrict__ pairs, int n,
                                                          long long frame_bytes) {
  const long long nvec = frame_bytes >> 4;
  const int per_frame = static_cast<int>((nvec + 8 * 256 - 1) / (8 * 256));  // rounds of 32 KB per frame
  const int total = per_frame * n;
  for (int w = blockIdx.x; w < total; w += gridDim.x) {
    const int f = w / per_frame, r = w - f * per_frame;
    const FramePair fp = pairs[f];
    const char* src = host + fp.src * frame_bytes;
    char* out = dev + fp.dst * frame_bytes;
    const long long j0 = static_cast<long long>(r) * 8 * 256 + threadIdx.x;
    uint4 val[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long j = j0 + u * 256;
      if (j < nvec) val[u] = ld_stream(src + j * 16);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long j = j0 + u * 256;
      if (j < nvec) st_stream(out + j * 16, val[u]);
    }
  }
}

// ---------------------------------------------------------------------------
// Decode snapshot: resolve each (member, block) of one layer's table row into
// a physical frame of the unified [pool | arena] buffer. GPU entries keep
// their slot id; CPU entries (encoded ~cpu_slot) point at the arena frame the
// prefetch writes: arena0 + member_base + b.
// Decode-time append (f2): one member's new token of one layer. Up to two
// destination frames (slot base addresses; host frames are mapped pinned
// memory written over the link), token row `tok` of every head's K and V.
struct AppendDesc {
  char* dst[2];
  int tok;
  int pad;
};

__global__ void append_kv_kernel(const AppendDesc* __restrict__ desc, const __nv_bfloat16* __restrict__ k,
                                 const __nv_bfloat16* __restrict__ v, int Hl, int bs, int D) {
  const AppendDesc a = desc[blockIdx.x];
  const int vec_per_row = D / 8;
  const int total = 2 * Hl * vec_per_row;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int c = i % vec_per_row;
    const int h = (i / vec_per_row) % Hl;
    const int kvsel = i / (vec_per_row * Hl);
    const __nv_bfloat16* src = (kvsel ? v : k) + (static_cast<long long>(blockIdx.x) * Hl + h) * D + c * 8;
    const uint4 val = *reinterpret_cast<const uint4*>(src);
    const long long off = ((static_cast<long long>(kvsel) * Hl + h) * bs + a.tok) * D * 2 + c * 16;
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (a.dst[j]) *reinterpret_cast<uint4*>(a.dst[j] + off) = val;
  }
}

struct SeqDesc {
  int row_offset;   // table offset of (row, layer 0, block 0)
  int kv_len;       // tokens attended
  int blk_offset;   // this member's first entry in the snapshot / arena
  int n_blocks;     // ceil(kv_len / bs)
};

__global__ void decode_snapshot_kernel(const int* __restrict__ table, const SeqDesc* __restrict__ seqs,
                                       int n_seq, int max_blocks, long long pool_frames,
                                       long long arena_frames, int depth, int* __restrict__ snap_all) {
  const int m = blockIdx.y, layer = blockIdx.z;
  if (m >= n_seq) return;
  const SeqDesc sd = seqs[m];
  const long long arena0 = pool_frames + (layer % depth) * arena_frames;
  int* snap = snap_all + layer * arena_frames;
  const int* row = table + sd.row_offset + static_cast<long long>(layer) * max_blocks;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < sd.n_blocks; b += gridDim.x * blockDim.x) {
    const int e = row[b];
    snap[sd.blk_offset + b] =
        e >= 0 ? e : static_cast<int>(arena0 + sd.blk_offset + b);
  }
}

// ---------------------------------------------------------------------------
// Synthetic data and verification.
__global__ void fill_kv_kernel(__nv_bfloat16* __restrict__ k, __nv_bfloat16* __restrict__ v,
                               long long tokens, long long token0, int layer, int Hl, int head0,
                               int D, unsigned long long seed) {
  const long long total = tokens * Hl * D;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int d = static_cast<int>(i % D);
    const int h = static_cast<int>((i / D) % Hl);
    const long long t = i / (static_cast<long long>(D) * Hl);
    const unsigned short kb = kv_value_bf16(seed, layer, 0, token0 + t, head0 + h, d);
    const unsigned short vb = kv_value_bf16(seed, layer, 1, token0 + t, head0 + h, d);
    reinterpret_cast<unsigned short*>(k)[i] = kb;
    reinterpret_cast<unsigned short*>(v)[i] = vb;
  }
}

// bf16 -> fp16, 8 values per thread step (the PF16 prefill attention's V
// copy). Exact for |x| in fp16's normal range [2^-14, 65504]; smaller values
// round to fp16 subnormals (absolute error <= 2^-25), larger ones SATURATE to
// +-65504 instead of becoming inf (which would turn whole output rows into
// NaN); NaN stays NaN. The input-range contract is stated on
// lkv_prefill_attention (include/lkv.h).
// The prefill attention is launched as its programmatic dependent: it loads
// Q and K and starts QK^T while this runs, and waits (griddepcontrol.wait)
// only before its first V load.
__device__ __forceinline__ float sat_f16(float x) {  // comparisons are false for NaN: it passes through
  return x > 65504.f ? 65504.f : (x < -65504.f ? -65504.f : x);
}

__global__ void bf16_to_f16_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, long long n8) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const uint4 a = __ldcs(src + i);
    const uint32_t w[4] = {a.x, a.y, a.z, a.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __half2 h = __floats2half2_rn(sat_f16(__uint_as_float(w[j] << 16)),
                                          sat_f16(__uint_as_float(w[j] & 0xFFFF0000u)));
      o[j] = *reinterpret_cast<const uint32_t*>(&h);
    }
    dst[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// Generator K/V of one token per row: row m holds token pos[m] of its own
// request (the decode step's new tokens).
__global__ void fill_kv_tokens_kernel(__nv_bfloat16* __restrict__ k, __nv_bfloat16* __restrict__ v,
                                      const long long* __restrict__ pos, int n, int layer, int Hl, int head0,
                                      int D, unsigned long long seed) {
  const long long total = static_cast<long long>(n) * Hl * D;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int d = static_cast<int>(i % D);
    const int h = static_cast<int>((i / D) % Hl);
    const long long t = pos[i / (static_cast<long long>(D) * Hl)];
    reinterpret_cast<unsigned short*>(k)[i] = kv_value_bf16(seed, layer, 0, t, head0 + h, d);
    reinterpret_cast<unsigned short*>(v)[i] = kv_value_bf16(seed, layer, 1, t, head0 + h, d);
  }
}

// One CTA per (block, layer) of a request: compare (or write) every element
// of the slot against the generator. The slot is found through the table
// mirror: GPU slot -> device pool, ~cpu_slot -> pinned host pool (read or
// written directly over the link).
template <bool kWrite>
__global__ void request_kv_kernel(const int* __restrict__ table_row, int max_blocks, int layer0,
                                  long long n_tokens, char* __restrict__ pool,
                                  char* __restrict__ host_pool, const int* __restrict__ xlat,
                                  long long slot_bytes, int Hl, int head0, int bs, int D,
                                  unsigned long long seed, unsigned long long* __restrict__ mismatches) {
  const int b = blockIdx.x, l = layer0 + static_cast<int>(blockIdx.y);
  const int e = table_row[static_cast<long long>(l) * max_blocks + b];
  // CPU slot ~e: its pinned frame (tiered host memory: through xlat)
  const long long hf = e >= 0 ? 0 : (xlat ? xlat[~e] : ~e);
  char* slot = e >= 0 ? pool + static_cast<long long>(e) * slot_bytes : host_pool + hf * slot_bytes;
  // 16 B per access: host frames are read/written over the link, where
  // narrow accesses would be transaction-bound.
  uint4* s128 = reinterpret_cast<uint4*>(slot);
  const int vec_row = D / 8;
  const int per_kv = Hl * bs * vec_row;
  unsigned long long bad = 0;
  for (int i = threadIdx.x; i < 2 * per_kv; i += blockDim.x) {
    const int kvsel = i / per_kv;
    int r = i % per_kv;
    const int d0 = (r % vec_row) * 8;
    r /= vec_row;
    const int t = r % bs;
    const int h = r / bs;
    const long long tok = static_cast<long long>(b) * bs + t;
    if (tok >= n_tokens) continue;
    unsigned w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      w[j] = static_cast<unsigned>(kv_value_bf16(seed, l, kvsel, tok, head0 + h, d0 + 2 * j)) |
             (static_cast<unsigned>(kv_value_bf16(seed, l, kvsel, tok, head0 + h, d0 + 2 * j + 1)) << 16);
    }
    if (kWrite) {
      s128[i] = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      const uint4 got = s128[i];
      bad += (got.x != w[0]) + (got.y != w[1]) + (got.z != w[2]) + (got.w != w[3]);
    }
  }
  if (!kWrite) {
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(mismatches, bad);
  }
}

}  // namespace lkv
