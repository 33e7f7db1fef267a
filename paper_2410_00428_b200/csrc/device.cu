// Device half of the LayerKV path (include/lkv.h "Device half").
//
// One lkv_device per GPU (per KV-head shard). It owns
//   * HBM: one buffer [pool frames | depth x arena frames] so that the decode
//     kernel addresses resident slots and prefetched frames uniformly; the
//     device block-table mirror; a decode snapshot; D2H staging segments;
//   * pinned host: the CPU slot pool (frame c = CPU slot c), a metadata
//     upload ring (journal, slot lists, descriptors);
//   * three streams: compute (table sync, scatter, pack, gather, attention),
//     d2h (offload copies), h2d (prefetch copies), ordered by events only.
// It is the KvManager's observer, so the reference call sequence (engine.cpp)
// drives the device path without new calls for escalation jobs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <deque>
#include <sstream>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include <cstdlib>

#include "decode_attn.cuh"
#include "decode_gqa_tc.cuh"
#include "prefill_attn2.cuh"
#include "host_mem.hpp"
#include "host_tier.hpp"
#include "kernels.cuh"
#include "layersim/errors.hpp"
#include "layersim/kv_manager.hpp"
#include "lkv.h"
#include "lkv_internal.hpp"

using layersim::KvManager;
using layersim::Loc;
using layersim::OffloadEntry;
using layersim::OffloadJob;
using layersim::RequestKv;


namespace lkv {

#define LKV_CUDA(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      throw CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_) + " (" __FILE__ \
                      ":" + std::to_string(__LINE__) + ")");                             \
    }                                                                                    \
  } while (0)

static int sm_count_of(int dev) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// Pinned ring for small host->device metadata. Regions are released once the
// event recorded after their consumer has completed.
class UploadRing {
 public:
  void init(std::size_t bytes) {
    LKV_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&buf_), bytes, cudaHostAllocMapped));
    cap_ = bytes;
  }
  void destroy() {
    for (auto& r : live_) cudaEventDestroy(r.ev);
    live_.clear();
    if (buf_) cudaFreeHost(buf_);
    buf_ = nullptr;
  }
  // Reserve `bytes` (16 B aligned); blocks on older consumers if needed.
  char* reserve(std::size_t bytes) {
    bytes = (bytes + 15) & ~std::size_t(15);
    if (bytes > cap_) throw CapacityError("upload ring: request larger than ring");
    if (head_ + bytes > cap_) head_ = 0;
    const std::size_t lo = head_, hi = head_ + bytes;
    // Retire in FIFO order until NO live region overlaps [lo, hi). After a
    // wrap the front can be an older region in the skipped tail while a
    // younger one at the ring's start overlaps, so checking only the front
    // is not enough.
    auto overlapping = [&] {
      for (const Region& r : live_)
        if (r.lo < hi && lo < r.hi) return true;
      return false;
    };
    while (!live_.empty()) {
      const Region& r = live_.front();
      if (live_.size() < 4096 && !overlapping()) break;
      LKV_CUDA(cudaEventSynchronize(r.ev));
      cudaEventDestroy(r.ev);
      live_.pop_front();
    }
    pending_lo_ = lo;
    pending_hi_ = hi;
    head_ = hi;
    return buf_ + lo;
  }
  // Mark the last reserved region in use by work already enqueued on `s`.
  void commit(cudaStream_t s) {
    cudaEvent_t ev;
    LKV_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    LKV_CUDA(cudaEventRecord(ev, s));
    live_.push_back({pending_lo_, pending_hi_, ev});
  }

 private:
  struct Region {
    std::size_t lo, hi;
    cudaEvent_t ev;
  };
  char* buf_ = nullptr;
  std::size_t cap_ = 0, head_ = 0, pending_lo_ = 0, pending_hi_ = 0;
  std::deque<Region> live_;
};

}  // namespace lkv

using namespace lkv;

struct lkv_device final : layersim::KvObserver {
  // ---- shape
  layersim::ModelSpec model;
  lkv_device_config cfg{};
  int L = 0, Hl = 0, Hql = 0, G = 0, D = 0, bs = 0, head0 = 0, sms = 148;
  long long sb = 0;  // slot bytes on this GPU
  long long seg_slots = 0;

  // ---- memory
  char* dbuf = nullptr;        // pool | arena stages
  char* host_pool = nullptr;   // pinned, CPU slot frames (tiered: the pinned frame tier)
  PinnedHost host_mem;         // host_pool's pages (untiered), on the GPU's NUMA node
  int numa_node = -1;          // the GPU's NUMA node (sysfs), -1 unknown
  // ---- tiered host memory: pageable homes + pinned frames
  HostTier tier;
  int* d_xlat = nullptr;        // [host_slots] CPU slot -> pinned frame (verify/fill kernels)
  FramePair* d_pull = nullptr;  // [arena_slots] (host frame, arena frame) list of one tiered prefetch
  bool tiered() const { return tier.enabled(); }
  // Frames of CPU slots for device access (identity when not tiered);
  // host_done() must follow once the work using them is enqueued on `st`.
  void host_frames(const std::vector<long long>& slots, bool read, std::vector<long long>* frames) {
    frames->resize(slots.size());
    if (!tiered()) {
      std::copy(slots.begin(), slots.end(), frames->begin());
      return;
    }
    if (!slots.empty()) tier.pin(slots.data(), static_cast<long long>(slots.size()), read, frames->data());
  }
  void host_done(const std::vector<long long>& slots, cudaStream_t st, bool write) {
    if (!tiered() || slots.empty()) return;
    cudaEvent_t ev;
    ev_create(&ev);
    LKV_CUDA(cudaEventRecord(ev, st));
    tier.used(slots.data(), static_cast<long long>(slots.size()), ev, write);  // takes the event
  }
  int* d_table = nullptr;      // [max_requests][L][max_blocks]
  unsigned* d_free_gpu = nullptr;   // free-list mirror (FreeSync): pushed part of the GPU stack, [gpu_slots]
  unsigned* d_free_cpu = nullptr;   // ... of the CPU stack, [host_slots]
  long long* d_free_hdr = nullptr;  // [2][3] {total, next_fresh, pushed size}
  bool free_full = true;            // next flush uploads both stacks whole (bind)
  int* d_snap = nullptr;       // [L][arena_slots]
  unsigned long long* d_stamps = nullptr;  // timing: [L][2] attention kernel span (%globaltimer min start, max end)
  unsigned long long* layer_stamps(int l) { return timing && d_stamps ? d_stamps + 2 * l : nullptr; }
  SeqDesc* d_seqs = nullptr;   // [max_batch]
  char* d_staging = nullptr;   // staging_chunks x seg bytes
  unsigned* d_slotlist = nullptr;  // staging_chunks x seg_slots GPU slot ids
  AttnSeq* d_aseqs = nullptr;      // [max_batch] (v2)
  AttnChunk* d_chunks = nullptr;   // chunk list of the iteration (v2)
  long long chunk_cap = 0, part_cap = 0;
  int n_chunks = 0;
  // Decode attention kernel by GQA group size: G = 1 the persistent CUDA-core
  // kernel fed by TMA bulk copies (decode_attn.cuh), G >= 2 the tcgen05 GQA
  // tile (decode_gqa_tc.cuh).
  bool tc_decode() const { return G >= 2; }
  // ---- fused all-gather of per-head outputs (decode_attn.cuh GatherArgs)
  char* d_gather = nullptr;                 // own gather buffer: flags | 2 parities of rows
  std::size_t gather_bytes = 0;
  std::vector<char*> gather_bases;          // per rank (own + IPC-opened or same-process peers)
  std::vector<char*> gather_opened;         // IPC mappings to close
  char** d_gather_bases = nullptr;
  unsigned* d_gather_done = nullptr;
  unsigned gather_epoch = 0;
  std::vector<unsigned> layer_epoch;        // [L] epoch of the layer's last gather
  bool gather_on() const { return d_gather_bases != nullptr; }
  long long gather_rows_per_parity() const { return static_cast<long long>(cfg.max_batch) * Hql * cfg.tp_size; }

  // fp16 copy of a prefill layer's V for the PF16 attention path
  void* d_vh = nullptr;
  std::size_t vh_cap = 0;
  cudaEvent_t vh_free = nullptr;
  bool vh_used = false;
  // Timing mode records no event between attention and merge: with the host
  // link saturated by the prefetch that event alone adds ~20 us per layer and
  // defeats programmatic dependent launch, so attn_ms covers the attention +
  // merge pair and merge_ms stays 0.
  CUtensorMap kvmap{};             // bf16 rows of 128 d over pool + arena frames, box {64, bs}
  float* d_part_o = nullptr;
  float* d_part_ml = nullptr;
  unsigned long long* d_counter = nullptr;
  UploadRing ring;
  static constexpr int kMaxSplits = 64;

  // ---- streams / events
  cudaStream_t cs = nullptr, d2h = nullptr, h2d = nullptr;
  std::vector<cudaEvent_t> seg_ready, seg_free;
  std::vector<char> seg_used;
  int seg_next = 0;
  std::vector<cudaEvent_t> fetch_done, attn_done;
  std::vector<char> attn_recorded;

  // ---- table mirror
  KvManager* kv = nullptr;
  std::unordered_map<long long, int> row_of;
  std::vector<int> free_rows;
  std::vector<TableUpdate> journal;

  // ---- offload bookkeeping
  std::unordered_map<long long, cudaEvent_t> job_ev;      // escalation job -> last copy
  std::unordered_map<long long, cudaEvent_t> prefill_ev;  // request -> last prefill D2H
  lkv_offload_stats ostats{};
  bool timing = false;
  cudaEvent_t t_pack0 = nullptr, t_pack1 = nullptr;

  // ---- decode iteration
  struct Member {
    long long id;
    int row, kv_len, nblk, blk_off;
    int fetch_len;  // cached tokens at decode_begin: what plan_decode_fetch books
  };
  bool append_mode = false;        // lkv_decode_begin_append: the step appends one token per member
  std::vector<char> appended;      // [L] append issued for the layer this iteration
  std::vector<Member> members;
  int total_blocks = 0, max_nblk = 0;
  bool in_iteration = false;
  lkv_decode_stats dstats{};
  std::vector<cudaEvent_t> t_attn0, t_attnk, t_attn1, t_f0, t_f1;  // per layer: attention | merge, prefetch copies
  std::vector<char> fetched;
  cudaEvent_t t_it0 = nullptr, t_it1 = nullptr, t_h2d0 = nullptr, t_h2d1 = nullptr;
  bool h2d_started = false;

  // ======================================================================
  void check_layer(int l) const {
    if (l < 0 || l >= L) throw std::invalid_argument("layer out of range");
  }

  static void ev_create(cudaEvent_t* e, bool timed = false) {
    LKV_CUDA(cudaEventCreateWithFlags(e, timed ? cudaEventDefault : cudaEventDisableTiming));
  }

  void init(const lkv_model_spec* m, int tpb, const lkv_device_config* c) {
    model = to_model(m);
    model.validate();
    cfg = *c;
    if (cfg.tp_size < 1 || cfg.tp_rank < 0 || cfg.tp_rank >= cfg.tp_size ||
        model.n_kv_heads % cfg.tp_size != 0)
      throw std::invalid_argument("tp_size must divide n_kv_heads and 0 <= tp_rank < tp_size");
    if (model.d_head != 128) throw std::invalid_argument("device path supports d_head = 128");
    if (model.f_precision != 2) throw std::invalid_argument("device path stores bf16 KV (f = 2)");
    if (tpb != 16 && tpb != 32 && tpb != 64)
      throw std::invalid_argument("tokens_per_block must be 16, 32 or 64");
    L = model.n_layers;
    D = model.d_head;
    bs = tpb;
    Hl = model.n_kv_heads / cfg.tp_size;
    G = model.n_heads / model.n_kv_heads;
    if (G * model.n_kv_heads != model.n_heads || (G != 1 && G != 2 && G != 4 && G != 8))
      throw std::invalid_argument("GQA group size must be 1, 2, 4 or 8");
    Hql = Hl * G;
    head0 = cfg.tp_rank * Hl;
    sb = 2ll * Hl * bs * D * 2;
    if (cfg.pipeline_depth < 1) cfg.pipeline_depth = 2;
    if (cfg.max_requests < 1 || cfg.max_blocks < 1 || cfg.max_batch < 1 || cfg.gpu_slots < 0 ||
        cfg.host_slots < 0 || cfg.arena_slots < 0)
      throw std::invalid_argument("device config sizes must be positive");
    if (cfg.staging_chunks < 2) cfg.staging_chunks = 4;
    if (cfg.chunk_bytes <= 0) cfg.chunk_bytes = 16ll << 20;
    seg_slots = std::max<long long>(1, cfg.chunk_bytes / sb);

    LKV_CUDA(cudaSetDevice(cfg.device));
    sms = sm_count_of(cfg.device);
    const long long frames = cfg.gpu_slots + cfg.arena_slots * cfg.pipeline_depth;
    if (frames > 0x7FFFFFFFll) throw CapacityError("pool + arena frames exceed int32 indexing");
    LKV_CUDA(cudaMalloc(&dbuf, std::max<long long>(frames, 1) * sb));

    numa_node = gpu_numa_node(cfg.device);
    const int cores = static_cast<int>(std::thread::hardware_concurrency());
    if (cfg.pinned_frames > 0 && cfg.host_slots > 0) {  // tiered: homes pageable, frames pinned
      // copy workers: the cores left beside the API and cleaner threads
      tier.init(cfg.device, cfg.host_slots, cfg.pinned_frames, sb, std::clamp(cores - 2, 2, 16), numa_node);
      host_pool = tier.pinned();
      LKV_CUDA(cudaMalloc(&d_xlat, cfg.host_slots * sizeof(int)));
      LKV_CUDA(cudaMalloc(&d_pull, std::max<long long>(cfg.arena_slots, 1) * sizeof(FramePair)));
    } else if (cfg.host_slots > 0) {
      host_mem.allocate(static_cast<std::size_t>(cfg.host_slots * sb), numa_node, std::clamp(cores, 1, 32));
      host_pool = host_mem.data();
    }
    const long long tbl = static_cast<long long>(cfg.max_requests) * L * cfg.max_blocks;
    // SeqDesc::row_offset and the snapshot kernel index the table in int32
    if (tbl > 0x7FFFFFFFll) throw CapacityError("max_requests x n_layers x max_blocks exceeds int32 table indexing");
    LKV_CUDA(cudaMalloc(&d_table, tbl * sizeof(int)));
    LKV_CUDA(cudaMalloc(&d_free_gpu, std::max<long long>(1, cfg.gpu_slots) * sizeof(unsigned)));
    LKV_CUDA(cudaMalloc(&d_free_cpu, std::max<long long>(1, cfg.host_slots) * sizeof(unsigned)));
    LKV_CUDA(cudaMalloc(&d_free_hdr, 6 * sizeof(long long)));
    LKV_CUDA(cudaMalloc(&d_snap, std::max<long long>(1, static_cast<long long>(L) * cfg.arena_slots) *
                                     sizeof(int)));
    LKV_CUDA(cudaMalloc(&d_seqs, cfg.max_batch * sizeof(SeqDesc)));
    LKV_CUDA(cudaMalloc(&d_staging, cfg.staging_chunks * seg_slots * sb));
    LKV_CUDA(cudaMalloc(&d_slotlist, cfg.staging_chunks * seg_slots * sizeof(unsigned)));
    // G >= 2: the group's QK^T / PV are dense enough that CUDA cores fall
    // behind HBM (32k x 16, scripts/attn_micro.py: v2 85/70/39% of peak at
    // G=2/4/8) -> tcgen05 tile (95/93/89%).
    {
      const unsigned long long rows = static_cast<unsigned long long>(std::max<long long>(frames, 1)) * 2 * Hl * bs;
      if (rows > 0x7FFFFFFFull) throw CapacityError("pool + arena rows exceed the TMA coordinate range");
      if (!tc::make_map_2d(&kvmap, dbuf, D, rows, static_cast<uint64_t>(D) * 2, 64, bs, true))
        throw CudaError("cuTensorMapEncodeTiled failed for the KV pool map");
    }
    LKV_CUDA(cudaMalloc(&d_aseqs, cfg.max_batch * sizeof(AttnSeq)));
    const long long parts = static_cast<long long>(cfg.max_batch) * Hql * kMaxSplits;
    part_cap = parts;
    LKV_CUDA(cudaMalloc(&d_part_o, parts * D * sizeof(float)));
    LKV_CUDA(cudaMalloc(&d_part_ml, parts * 2 * sizeof(float)));
    LKV_CUDA(cudaMalloc(&d_counter, sizeof(unsigned long long)));
    ring.init(64ull << 20);

    LKV_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    LKV_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    LKV_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    // Attention reads whole blocks and masks the tail; never let a tail be an
    // uninitialised NaN pattern (0 * NaN poisons P.V). Ordered on the compute
    // stream (a legacy-stream memset would race the non-blocking streams).
    LKV_CUDA(cudaMemsetAsync(dbuf, 0, std::max<long long>(frames, 1) * sb, cs));
    LKV_CUDA(cudaMemsetAsync(d_table, 0, tbl * sizeof(int), cs));
    LKV_CUDA(cudaMemsetAsync(d_free_hdr, 0, 6 * sizeof(long long), cs));
    LKV_CUDA(cudaStreamSynchronize(cs));
    seg_ready.resize(cfg.staging_chunks);
    seg_free.resize(cfg.staging_chunks);
    seg_used.assign(cfg.staging_chunks, 0);
    for (int i = 0; i < cfg.staging_chunks; ++i) {
      ev_create(&seg_ready[i]);
      ev_create(&seg_free[i]);
    }
    fetch_done.resize(cfg.pipeline_depth);
    attn_done.resize(cfg.pipeline_depth);
    attn_recorded.assign(cfg.pipeline_depth, 0);
    for (int i = 0; i < cfg.pipeline_depth; ++i) {
      ev_create(&fetch_done[i]);
      ev_create(&attn_done[i]);
    }
    t_attn0.resize(L);
    t_attnk.resize(L);
    t_attn1.resize(L);
    t_f0.resize(L);
    t_f1.resize(L);
    fetched.assign(L, 0);
    for (int i = 0; i < L; ++i) {
      ev_create(&t_attn0[i], true);
      ev_create(&t_attnk[i], true);
      ev_create(&t_attn1[i], true);
      ev_create(&t_f0[i], true);
      ev_create(&t_f1[i], true);
    }
    ev_create(&t_it0, true);
    ev_create(&t_it1, true);
    ev_create(&t_h2d0, true);
    ev_create(&t_h2d1, true);
    ev_create(&t_pack0, true);
    ev_create(&t_pack1, true);
    ev_create(&ev_join);
    ev_create(&vh_free);
    for (int r = cfg.max_requests - 1; r >= 0; --r) free_rows.push_back(r);
  }

  ~lkv_device() override {
    if (kv) kv->set_observer(nullptr);
    cudaSetDevice(cfg.device);
    if (cs) cudaStreamSynchronize(cs);
    if (d2h) cudaStreamSynchronize(d2h);
    if (h2d) cudaStreamSynchronize(h2d);
    auto kill = [](std::vector<cudaEvent_t>& v) {
      for (auto e : v)
        if (e) cudaEventDestroy(e);
    };
    kill(seg_ready);
    kill(seg_free);
    kill(fetch_done);
    kill(attn_done);
    kill(t_attn0);
    kill(t_attnk);
    kill(t_attn1);
    kill(t_f0);
    kill(t_f1);
    drain_timed(d2h_timed);
    for (auto e : {t_it0, t_it1, t_h2d0, t_h2d1, t_pack0, t_pack1, ev_join})
      if (e) cudaEventDestroy(e);
    for (auto& kvp : job_ev) cudaEventDestroy(kvp.second);
    for (auto& kvp : prefill_ev) cudaEventDestroy(kvp.second);
    ring.destroy();
    cudaFree(dbuf);
    host_mem.release();
    tier.destroy();
    cudaFree(d_xlat);
    cudaFree(d_pull);
    cudaFree(d_table);
    cudaFree(d_free_gpu);
    cudaFree(d_free_cpu);
    cudaFree(d_free_hdr);
    cudaFree(d_snap);
    cudaFree(d_stamps);
    cudaFree(d_seqs);
    cudaFree(d_staging);
    cudaFree(d_slotlist);
    cudaFree(d_part_o);
    cudaFree(d_part_ml);
    cudaFree(d_aseqs);
    cudaFree(d_chunks);
    cudaFree(d_counter);
    cudaFree(d_vh);
    if (vh_free) cudaEventDestroy(vh_free);
    for (char* p : gather_opened) cudaIpcCloseMemHandle(p);
    cudaFree(d_gather);
    cudaFree(d_gather_bases);
    cudaFree(d_gather_done);
    for (auto s : {cs, d2h, h2d})
      if (s) cudaStreamDestroy(s);
  }

  // ---------------------------------------------------------------- table
  static int enc(const layersim::SlotLoc& e) {
    if (e.loc == Loc::Gpu) return static_cast<int>(e.slot);
    if (e.loc == Loc::Cpu) return ~static_cast<int>(e.slot);
    return ~0x7FFFFFFF;
  }
  long long tindex(int row, int l, int b) const {
    return (static_cast<long long>(row) * L + l) * cfg.max_blocks + b;
  }
  void check_slot(const layersim::SlotLoc& e) const {
    if (e.loc == Loc::Gpu && static_cast<long long>(e.slot) >= cfg.gpu_slots)
      throw CapacityError("GPU slot " + std::to_string(e.slot) + " >= device pool frames " +
                          std::to_string(cfg.gpu_slots));
    if (e.loc == Loc::Cpu && static_cast<long long>(e.slot) >= cfg.host_slots)
      throw CapacityError("CPU slot " + std::to_string(e.slot) + " >= pinned host frames " +
                          std::to_string(cfg.host_slots));
  }

  // The journal may update one table entry several times before a flush
  // (e.g. complete_offload rewrites a row, release frees it, allocate_prefill
  // hands it to the next request). table_apply_kernel writes in parallel, so
  // only the last update per entry is kept (in journal order).
  std::unordered_map<long long, std::size_t> journal_last;
  void dedupe_journal() {
    journal_last.clear();
    journal_last.reserve(journal.size() * 2);
    bool dup = false;
    for (std::size_t i = 0; i < journal.size(); ++i) {
      auto [it, fresh] = journal_last.try_emplace(journal[i].index, i);
      if (!fresh) {
        it->second = i;
        dup = true;
      }
    }
    if (!dup) return;
    std::size_t w = 0;
    for (std::size_t i = 0; i < journal.size(); ++i)
      if (journal_last[journal[i].index] == i) journal[w++] = journal[i];
    journal.resize(w);
  }

  // Applies the table journal and the free lists' changes (the device mirror
  // of the manager's state) with one kernel on the
  // compute stream, ahead of any consumer.
  void flush() {
    FreeSync fs{};
    KvManager::FreeListDelta fd[2];
    if (kv) {
      for (int l = 0; l < 2; ++l) {
        fd[l] = kv->take_free_delta(l == 0, free_full);
        const long long cap = l == 0 ? cfg.gpu_slots : cfg.host_slots;
        if (fd[l].size > cap)
          throw CapacityError("device free-list mirror: " + std::to_string(fd[l].size) + " free " +
                              (l == 0 ? "GPU" : "CPU") + " slots > " + std::to_string(cap) + " frames");
        if (fd[l].changed) fs.any = 1;
      }
      free_full = false;
    }
    if (journal.empty() && !fs.any) return;
    dedupe_journal();
    const std::size_t n = journal.size();
    const std::size_t tbytes = (n * sizeof(TableUpdate) + 15) & ~std::size_t(15);
    std::size_t fbytes[2] = {0, 0};
    if (fs.any)
      for (int l = 0; l < 2; ++l) fbytes[l] = ((fd[l].size - fd[l].low) * sizeof(unsigned) + 15) & ~std::size_t(15);
    char* up = ring.reserve(std::max<std::size_t>(16, tbytes + fbytes[0] + fbytes[1]));
    auto* dst = reinterpret_cast<TableUpdate*>(up);
    if (n) std::memcpy(dst, journal.data(), n * sizeof(TableUpdate));
    long long work = static_cast<long long>(n);
    if (fs.any) {
      char* p = up + tbytes;
      for (int l = 0; l < 2; ++l) {
        const long long cnt = fd[l].size - fd[l].low;
        if (cnt) std::memcpy(p, fd[l].pushed + fd[l].low, cnt * sizeof(unsigned));
        fs.src[l] = reinterpret_cast<const unsigned*>(p);
        fs.dst[l] = l == 0 ? d_free_gpu : d_free_cpu;
        fs.low[l] = fd[l].low;
        fs.n[l] = cnt;
        fs.total[l] = l == 0 ? kv->gpu_blocks_total() : kv->cpu_blocks_total();
        fs.fresh[l] = fd[l].next_fresh;
        fs.size[l] = fd[l].size;
        work = std::max(work, cnt);
        p += fbytes[l];
      }
      fs.hdr = d_free_hdr;
    }
    const int threads = 256;
    const int grid = static_cast<int>(std::clamp<long long>((work + threads - 1) / threads, 1, 4ll * sms));
    table_apply_kernel<<<grid, threads, 0, cs>>>(dst, static_cast<int>(n), d_table, fs);
    LKV_CUDA(cudaGetLastError());
    ring.commit(cs);
    journal.clear();
  }

  int row_for(long long id) const {
    auto it = row_of.find(id);
    if (it == row_of.end()) throw layersim::SimulationError("device: request " + std::to_string(id) + " has no table row");
    return it->second;
  }

  void on_allocate(std::int64_t id, const RequestKv& r) override {
    if (free_rows.empty()) throw CapacityError("device: all block-table rows in use");
    if (static_cast<long long>(r.blocks.size()) > cfg.max_blocks)
      throw CapacityError("device: request exceeds max_blocks per table row");
    const int row = free_rows.back();
    free_rows.pop_back();
    row_of[id] = row;
    journal.reserve(journal.size() + r.blocks.size() * L);
    for (std::size_t b = 0; b < r.blocks.size(); ++b)
      for (int l = 0; l < L; ++l) {
        const auto& e = r.blocks[b].layers[l];
        check_slot(e);
        journal.push_back({tindex(row, l, static_cast<int>(b)), enc(e), 0});
      }
  }

  void on_append(std::int64_t id, const RequestKv& r) override {
    const int row = row_for(id);
    const int b = static_cast<int>(r.blocks.size()) - 1;
    if (b >= cfg.max_blocks) throw CapacityError("device: request exceeds max_blocks per table row");
    for (int l = 0; l < L; ++l) {
      const auto& e = r.blocks[b].layers[l];
      check_slot(e);
      journal.push_back({tindex(row, l, b), enc(e), 0});
    }
  }

  void on_manager_destroyed() override { kv = nullptr; }

  void on_release(std::int64_t id, const RequestKv& r) override {
    if (tiered()) {  // the request's CPU slots return to the pool: drop their frames, no write-back
      std::vector<long long> dead;
      for (const auto& blk : r.blocks)
        for (const auto& e : blk.layers)
          if (e.loc == Loc::Cpu) dead.push_back(e.slot);
      tier.forget(dead.data(), static_cast<long long>(dead.size()));
    }
    auto it = row_of.find(id);
    if (it == row_of.end()) return;
    free_rows.push_back(it->second);
    row_of.erase(it);
    // Freed CPU frames may be rewritten by a later D2H: order those copies
    // after every prefetch already reading them.
    cudaEvent_t ev;
    ev_create(&ev);
    LKV_CUDA(cudaEventRecord(ev, h2d));
    LKV_CUDA(cudaStreamWaitEvent(d2h, ev, 0));
    cudaEventDestroy(ev);
    auto pe = prefill_ev.find(id);
    if (pe != prefill_ev.end()) {
      cudaEventDestroy(pe->second);
      prefill_ev.erase(pe);
    }
  }

  // ------------------------------------------------------- D2H staging pipeline
  // Copy `n` frames between a contiguous side and an arbitrary frame list,
  // coalescing runs of constant positive stride into one 2D copy each.
  int emit_copies(char* dst_base, const long long* dst_frames, const char* src_base,
                  const long long* src_frames, long long n, cudaMemcpyKind kind,
                  cudaStream_t s) {
    int copies = 0;
    long long i = 0;
    while (i < n) {
      long long j = i + 1;
      long long dd = 0, ds = 0;
      if (j < n) {
        dd = dst_frames[j] - dst_frames[i];
        ds = src_frames[j] - src_frames[i];
        if (dd > 0 && ds > 0) {
          while (j + 1 < n && dst_frames[j + 1] - dst_frames[j] == dd &&
                 src_frames[j + 1] - src_frames[j] == ds)
            ++j;
          ++j;
        } else {
          j = i + 1;
        }
      }
      const long long len = j - i;
      char* d = dst_base + dst_frames[i] * sb;
      const char* sp = src_base + src_frames[i] * sb;
      if (len == 1 || (dd == 1 && ds == 1)) {  // contiguous: one linear copy (batched below)
        b_dst.push_back(d);
        b_src.push_back(const_cast<char*>(sp));
        b_size.push_back(static_cast<std::size_t>(len * sb));
      } else {
        LKV_CUDA(cudaMemcpy2DAsync(d, dd * sb, sp, ds * sb, sb, len, kind, s));
        ++copies;
      }
      i = j;
    }
    copies += flush_linear(kind, s);
    return copies;
  }

  // Linear copies of one emit_copies call, one cudaMemcpyAsync each (the
  // batched-copy API is closed on this pool: it raised GPU faults). Tiered
  // frames are handed out in ascending order, so runs coalesce before this.
  std::vector<void*> b_dst, b_src;
  std::vector<std::size_t> b_size;
  int flush_linear(cudaMemcpyKind kind, cudaStream_t s) {
    const std::size_t n = b_dst.size();
    for (std::size_t k = 0; k < n; ++k) LKV_CUDA(cudaMemcpyAsync(b_dst[k], b_src[k], b_size[k], kind, s));
    const int copies = static_cast<int>(n);
    b_dst.clear();
    b_src.clear();
    b_size.clear();
    return copies;
  }

  // Scatter K/V blocks [b0, b0+n) of a prefill layer into slots: frames =
  // the layer's table row (GPU slots, absolute block index) or nullptr for a
  // contiguous destination (staging).
  void scatter_blocks(const __nv_bfloat16* kb, const __nv_bfloat16* vb, long long tokens, long long b0, long long n,
                      const int* frames, char* dst, bool reverse = false) {
    if (n <= 0) return;
    // D = 128 and bs in {16, 32, 64} (init): one CTA per K or V half slot
    scatter_slots_kernel<<<static_cast<unsigned>(2 * n), 256, 0, cs>>>(kb, vb, tokens, static_cast<int>(b0), frames,
                                                                      dst, sb, Hl, __builtin_ctz(bs),
                                                                      reverse ? static_cast<int>(n) : 0);
    LKV_CUDA(cudaGetLastError());
  }

  int next_segment() {
    const int i = seg_next;
    seg_next = (seg_next + 1) % cfg.staging_chunks;
    if (seg_used[i]) LKV_CUDA(cudaStreamWaitEvent(cs, seg_free[i], 0));
    seg_used[i] = 1;
    return i;
  }

  // Stream frames [i0, i0+n) of a staging producer to host frames cpu[...].
  // Copy-engine busy time (timing on): event pairs around each batch of
  // copies on a copy stream, summed when the stats are read.
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> d2h_timed;
  void timed_begin(cudaStream_t st, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
    cudaEvent_t a, b;
    ev_create(&a, true);
    ev_create(&b, true);
    LKV_CUDA(cudaEventRecord(a, st));
    v.push_back({a, b});
  }
  void timed_end(cudaStream_t st, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
    LKV_CUDA(cudaEventRecord(v.back().second, st));
  }
  static double drain_timed(std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
    double ms = 0.0;
    for (auto& pr : v) {
      float t = 0.f;
      if (cudaEventSynchronize(pr.second) == cudaSuccess && cudaEventElapsedTime(&t, pr.first, pr.second) == cudaSuccess)
        ms += t;
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
    cudaGetLastError();
    v.clear();
    return ms;
  }

  void d2h_segment(int seg, const long long* cpu_slots, long long n) {
    LKV_CUDA(cudaEventRecord(seg_ready[seg], cs));
    LKV_CUDA(cudaStreamWaitEvent(d2h, seg_ready[seg], 0));
    std::vector<long long> src(n), slots(cpu_slots, cpu_slots + n), frames;
    for (long long i = 0; i < n; ++i) src[i] = seg * seg_slots + i;
    host_frames(slots, false, &frames);  // whole frames are overwritten: no read-in
    if (timing) timed_begin(d2h, d2h_timed);
    ostats.d2h_copies +=
        emit_copies(host_pool, frames.data(), d_staging, src.data(), n, cudaMemcpyDeviceToHost, d2h);
    if (timing) timed_end(d2h, d2h_timed);
    host_done(slots, d2h, true);
    ostats.d2h_bytes_physical += n * sb;
    LKV_CUDA(cudaEventRecord(seg_free[seg], d2h));
  }

  void on_offload_planned(const OffloadJob& job, const std::vector<OffloadEntry>& entries) override {
    flush();
    const long long n = static_cast<long long>(entries.size());
    long long tokens = 0;
    for (const auto& e : entries) {
      if (static_cast<long long>(e.cpu_slot) >= cfg.host_slots)
        throw CapacityError("CPU slot " + std::to_string(e.cpu_slot) + " >= host frames");
      tokens += e.filled_tokens;
    }
    // Staging order = ascending CPU slot (the gather takes any GPU slot
    // order), so runs of destination frames coalesce into single copies.
    std::vector<long long> ord(static_cast<std::size_t>(n));
    for (long long i = 0; i < n; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(),
                     [&](long long a, long long b) { return entries[a].cpu_slot < entries[b].cpu_slot; });
    // One gather launch per run of consecutive staging segments (up to the
    // ring's wrap; a CTA per slot), then one D2H per segment.
    long long i0 = 0;
    while (i0 < n) {
      const long long want = (n - i0 + seg_slots - 1) / seg_slots;
      const long long nseg = std::min<long long>(want, cfg.staging_chunks - seg_next);
      const int seg0 = seg_next;
      for (long long k = 0; k < nseg; ++k) next_segment();
      const long long cnt_all = std::min(nseg * seg_slots, n - i0);
      auto* slots = reinterpret_cast<unsigned*>(ring.reserve(cnt_all * sizeof(unsigned)));
      for (long long i = 0; i < cnt_all; ++i) slots[i] = entries[ord[i0 + i]].gpu_slot;
      unsigned* dl = d_slotlist + seg0 * seg_slots;
      LKV_CUDA(cudaMemcpyAsync(dl, slots, cnt_all * sizeof(unsigned), cudaMemcpyHostToDevice, cs));
      ring.commit(cs);
      gather_slots_v2_kernel<<<static_cast<unsigned>(cnt_all), 256, 0, cs>>>(dbuf, dl, sb,
                                                                              d_staging + seg0 * seg_slots * sb);
      LKV_CUDA(cudaGetLastError());
      for (long long k = 0; k < nseg; ++k) {
        const long long s0 = i0 + k * seg_slots;
        const long long cnt = std::min(seg_slots, n - s0);
        std::vector<long long> cpu(cnt);
        for (long long i = 0; i < cnt; ++i) cpu[i] = entries[ord[s0 + i]].cpu_slot;
        d2h_segment(seg0 + static_cast<int>(k), cpu.data(), cnt);
      }
      i0 += cnt_all;
    }
    cudaEvent_t ev;
    ev_create(&ev, true);
    LKV_CUDA(cudaEventRecord(ev, d2h));
    job_ev[job.job_id] = ev;
    ostats.jobs += 1;
    ostats.d2h_bytes_algorithmic += tokens * (sb / bs);
  }

  void on_offload_complete(std::int64_t job_id, std::int64_t rid, bool orphaned,
                           const RequestKv*) override {
    auto it = job_ev.find(job_id);
    if (it != job_ev.end()) {
      LKV_CUDA(cudaEventSynchronize(it->second));  // send buffers drained
      cudaEventDestroy(it->second);
      job_ev.erase(it);
    }
    if (orphaned) {  // the reserved CPU destinations return to the pool: their bytes are dead
      if (tiered()) {
        std::vector<long long> dead;
        for (const auto& e : kv->offload_entries(job_id)) dead.push_back(e.cpu_slot);
        tier.forget(dead.data(), static_cast<long long>(dead.size()));
      }
      return;
    }
    const int row = row_for(rid);
    for (const auto& e : kv->offload_entries(job_id))
      journal.push_back({tindex(row, e.layer, e.block), ~static_cast<int>(e.cpu_slot), 0});
  }

  // ---------------------------------------------------------------- prefill
  // Ordering with a caller's stream: inputs produced on `user` are read on the
  // compute stream only after join_in; the caller's later work (reusing the
  // inputs, reading outputs) waits for the compute stream after join_out.
  cudaEvent_t ev_join = nullptr;
  void join_in(cudaStream_t user) {
    if (!user || user == cs) return;
    LKV_CUDA(cudaEventRecord(ev_join, user));
    LKV_CUDA(cudaStreamWaitEvent(cs, ev_join, 0));
  }
  void join_out(cudaStream_t user) {
    if (!user || user == cs) return;
    LKV_CUDA(cudaEventRecord(ev_join, cs));
    LKV_CUDA(cudaStreamWaitEvent(user, ev_join, 0));
  }

  void prefill_layer(long long id, int l, const void* k, const void* v, long long tokens,
                     cudaStream_t user) {
    check_layer(l);
    flush();
    join_in(user);
    const RequestKv& r = kv->request(id);
    const int row = row_for(id);
    const long long nb = std::min<long long>((tokens + bs - 1) / bs, static_cast<long long>(r.blocks.size()));
    if (tokens > static_cast<long long>(r.blocks.size()) * bs)
      throw std::invalid_argument("prefill_layer: more tokens than allocated blocks");
    if (timing) LKV_CUDA(cudaEventRecord(t_pack0, cs));
    // GPU-resident blocks: scatter through the table mirror (CPU entries skipped).
    long long n_gpu = 0;
    for (long long b = 0; b < nb; ++b) n_gpu += r.blocks[b].layers[l].loc == Loc::Gpu;
    const auto* kb = static_cast<const __nv_bfloat16*>(k);
    const auto* vb = static_cast<const __nv_bfloat16*>(v);
    if (n_gpu == nb && nb > 0) {
      scatter_blocks(kb, vb, tokens, 0, nb, d_table + tindex(row, l, 0), dbuf);
      ostats.scatter_bytes += nb * sb;
    } else {
      // Runs of blocks by residency; GPU runs scatter, CPU runs pack+D2H.
      long long b = 0;
      while (b < nb) {
        const Loc where = r.blocks[b].layers[l].loc;
        long long e = b + 1;
        while (e < nb && r.blocks[e].layers[l].loc == where) ++e;
        if (where == Loc::Gpu) {
          scatter_blocks(kb, vb, tokens, b, e - b, d_table + tindex(row, l, 0), dbuf);
          ostats.scatter_bytes += (e - b) * sb;
        } else if (where == Loc::Cpu) {
          // One pack launch per run of consecutive staging segments (up to the
          // ring's wrap), then one D2H per segment.
          long long c0 = b;
          while (c0 < e) {
            const long long want = (e - c0 + seg_slots - 1) / seg_slots;
            const long long nseg = std::min<long long>(want, cfg.staging_chunks - seg_next);
            const int seg0 = seg_next;
            for (long long k = 0; k < nseg; ++k) next_segment();
            const long long cnt_all = std::min(nseg * seg_slots, e - c0);
            std::vector<long long> cpu(cnt_all);
            for (long long i = 0; i < cnt_all; ++i) {
              const auto& en = r.blocks[c0 + i].layers[l];
              check_slot(en);
              cpu[i] = en.slot;
            }
            // block c0 + i -> staging slot i; a span whose CPU slots descend
            // (a released request's slots popped back off the LIFO list) is
            // packed in reverse, so staging and host frames ascend together
            const bool rev = cnt_all > 1 && cpu.front() > cpu.back();
            if (rev) std::reverse(cpu.begin(), cpu.end());
            scatter_blocks(kb, vb, tokens, c0, cnt_all, nullptr, d_staging + seg0 * seg_slots * sb, rev);
            for (long long k = 0; k < nseg; ++k) {
              const long long p0 = k * seg_slots;
              const long long cnt = std::min(seg_slots, cnt_all - p0);
              if (cnt <= 0) break;
              d2h_segment(seg0 + static_cast<int>(k), cpu.data() + p0, cnt);
            }
            const long long tok_hi = std::min(tokens, (c0 + cnt_all) * bs);
            ostats.d2h_bytes_algorithmic += (tok_hi - c0 * bs) * (sb / bs);
            c0 += cnt_all;
          }
        }
        b = e;
      }
      cudaEvent_t& ev = prefill_ev[id];
      if (!ev) ev_create(&ev);
      LKV_CUDA(cudaEventRecord(ev, d2h));
    }
    if (timing) LKV_CUDA(cudaEventRecord(t_pack1, cs));
    join_out(user);  // k/v may be overwritten once the scatter/pack has read them
  }

  // ----------------------------------------------------------------- decode
  // Layer l's prefetch: every member's CPU-located blocks (blocks past the
  // member's fetch length are the appended token's fresh block), their arena
  // frames, and the token-exact bytes plan_decode_fetch books for them.
  struct FetchPlan {
    std::vector<long long> slots, dst;
    std::vector<std::size_t> first;  // [members + 1] member ranges in slots / dst
    long long tokens = 0;
  };
  FetchPlan fetch_plan(int l) const {
    FetchPlan p;
    const int st = l % cfg.pipeline_depth;
    const long long arena0 = cfg.gpu_slots + static_cast<long long>(st) * cfg.arena_slots;
    p.first.assign(members.size() + 1, 0);
    for (std::size_t mi = 0; mi < members.size(); ++mi) {
      const Member& m = members[mi];
      const RequestKv& r = kv->request(m.id);
      for (int b = 0; b < m.nblk; ++b) {
        if (static_cast<long long>(b) * bs >= m.fetch_len) break;
        const auto& e = r.blocks[b].layers[l];
        if (e.loc != Loc::Cpu) continue;
        check_slot(e);
        p.slots.push_back(e.slot);
        p.dst.push_back(arena0 + m.blk_off + b);
        p.tokens += std::clamp<long long>(m.fetch_len - static_cast<long long>(b) * bs, 0, bs);
      }
      p.first[mi + 1] = p.slots.size();
    }
    return p;
  }

  // Tiered host memory: layers whose read-ins were started ahead of their
  // prefetch (HostTier::stage), `read_ahead` layers beyond the one issued.
  int read_ahead = 0;
  std::vector<std::vector<long long>> staged_slots;  // [L] slots staged, not yet pinned
  std::vector<char> staged;                          // [L]
  void stage_layer(int l) {
    if (!tiered() || l >= L || staged[l]) return;
    staged[l] = 1;
    staged_slots[l] = fetch_plan(l).slots;
    if (!staged_slots[l].empty()) tier.stage(staged_slots[l].data(), static_cast<long long>(staged_slots[l].size()));
  }

  void issue_fetch(int l) {
    const int st = l % cfg.pipeline_depth;
    if (attn_recorded[st]) LKV_CUDA(cudaStreamWaitEvent(h2d, attn_done[st], 0));
    if (timing && !h2d_started) {
      LKV_CUDA(cudaEventRecord(t_h2d0, h2d));
      h2d_started = true;
    }
    const long long copies0 = dstats.h2d_copies;
    if (timing) LKV_CUDA(cudaEventRecord(t_f0[l], h2d));
    FetchPlan p = fetch_plan(l);
    dstats.h2d_bytes_algorithmic += p.tokens * (sb / bs);
    std::vector<long long> all_frames;
    host_frames(p.slots, true, &all_frames);  // tiered: staged read-ins landed / missing slots read in
    if (tiered() && l < L) {
      staged[l] = 1;  // its stage locks became the pin's locks
      staged_slots[l].clear();
    }
    if (tiered()) {
      // the tier's frames of a layer are scattered (LRU order): one pull
      // kernel over the link instead of one copy-engine transfer per frame
      const long long n = static_cast<long long>(all_frames.size());
      if (n > 0) {
        auto* pairs = reinterpret_cast<FramePair*>(ring.reserve(n * sizeof(FramePair)));
        for (long long i = 0; i < n; ++i) pairs[i] = {all_frames[i], p.dst[i]};
        LKV_CUDA(cudaMemcpyAsync(d_pull, pairs, n * sizeof(FramePair), cudaMemcpyHostToDevice, h2d));
        ring.commit(h2d);
        const long long rounds = n * ((sb / 16 + 2047) / 2048);
        const int grid = static_cast<int>(std::min<long long>(rounds, std::max(sms / 2, 1)));
        pull_frames_kernel<<<grid, 256, 0, h2d>>>(host_pool, dbuf, d_pull, static_cast<int>(n), sb);
        LKV_CUDA(cudaGetLastError());
        dstats.kernel_launches += 1;
        dstats.h2d_copies += 1;
        dstats.h2d_bytes_physical += n * sb;
      }
    } else {
      for (std::size_t mi = 0; mi < members.size(); ++mi) {
        const std::size_t a = p.first[mi], n = p.first[mi + 1] - a;
        if (n == 0) continue;
        dstats.h2d_copies += emit_copies(dbuf, p.dst.data() + a, host_pool, all_frames.data() + a,
                                         static_cast<long long>(n), cudaMemcpyHostToDevice, h2d);
        dstats.h2d_bytes_physical += static_cast<long long>(n) * sb;
      }
    }
    host_done(p.slots, h2d, false);
    LKV_CUDA(cudaEventRecord(fetch_done[st], h2d));
    if (timing) {
      LKV_CUDA(cudaEventRecord(t_f1[l], h2d));
      fetched[l] = dstats.h2d_copies > copies0;
      LKV_CUDA(cudaEventRecord(t_h2d1, h2d));
    }
    stage_layer(l + read_ahead);  // keep the read-ins `read_ahead` layers ahead of the DMA
  }

  void decode_begin(const int64_t* ids, int n, bool append = false) {
    if (in_iteration) throw layersim::SimulationError("decode_begin: iteration already open");
    append_mode = append;
    appended.assign(L, 0);
    fetched.assign(L, 0);
    if (n < 0 || n > cfg.max_batch) throw CapacityError("decode batch exceeds max_batch");
    flush();
    members.clear();
    total_blocks = 0;
    max_nblk = 0;
    dstats = lkv_decode_stats{};
    h2d_started = false;
    auto* desc = reinterpret_cast<SeqDesc*>(ring.reserve(std::max(n, 1) * sizeof(SeqDesc)));
    for (int i = 0; i < n; ++i) {
      const RequestKv& r = kv->request(ids[i]);
      Member m;
      m.id = ids[i];
      m.row = row_for(ids[i]);
      m.fetch_len = static_cast<int>(r.cached_tokens);
      m.kv_len = m.fetch_len + (append ? 1 : 0);
      if (append && static_cast<long long>(r.blocks.size()) * bs < m.kv_len)
        throw layersim::SimulationError("decode append: request " + std::to_string(ids[i]) +
                                        " has no block for its next token (append_decode_block first)");
      m.nblk = static_cast<int>(std::min<long long>((m.kv_len + bs - 1) / bs, static_cast<long long>(r.blocks.size())));
      m.blk_off = total_blocks;
      total_blocks += m.nblk;
      max_nblk = std::max(max_nblk, m.nblk);
      members.push_back(m);
      desc[i] = {static_cast<int>(tindex(m.row, 0, 0)), m.kv_len, m.blk_off, m.nblk};
      dstats.kv_bytes_read += static_cast<long long>(m.kv_len) * (sb / bs) * L;
    }
    if (total_blocks > cfg.arena_slots)
      throw CapacityError("decode batch needs " + std::to_string(total_blocks) +
                          " arena frames per stage, have " + std::to_string(cfg.arena_slots));
    if (timing) LKV_CUDA(cudaEventRecord(t_it0, cs));
    LKV_CUDA(cudaMemcpyAsync(d_seqs, desc, std::max(n, 1) * sizeof(SeqDesc), cudaMemcpyHostToDevice, cs));
    ring.commit(cs);
    plan_chunks();
    if (n > 0 && max_nblk > 0) {
      // one launch resolves every layer; layer l's arena stage is l % depth
      dim3 grid((max_nblk + 255) / 256, n, L);
      dstats.kernel_launches += 1;
      decode_snapshot_kernel<<<grid, 256, 0, cs>>>(d_table, d_seqs, n, cfg.max_blocks, cfg.gpu_slots,
                                                   cfg.arena_slots, cfg.pipeline_depth, d_snap);
      LKV_CUDA(cudaGetLastError());
    }
    // A member's prefetch reads CPU frames its own prefill offload may still
    // be writing: wait for that request's last prefill D2H only. Escalation
    // jobs need no wait (their entries stay GPU-located until
    // complete_offload, which synchronises the job's copies first), so the
    // D2H and H2D engines keep running concurrently (full duplex).
    for (const Member& m : members) {
      auto pe = prefill_ev.find(m.id);
      if (pe != prefill_ev.end()) LKV_CUDA(cudaStreamWaitEvent(h2d, pe->second, 0));
    }
    if (timing) {
      if (!d_stamps) LKV_CUDA(cudaMalloc(&d_stamps, static_cast<std::size_t>(std::max(L, 1)) * 16));
      LKV_CUDA(cudaMemsetAsync(d_stamps, 0, static_cast<std::size_t>(std::max(L, 1)) * 16, cs));
    }
    in_iteration = true;
    if (tiered()) {
      // read-ahead depth: the layers staged ahead take their frames from the
      // least recently used ones, which must already be past their DMA — a
      // victim still in flight blocks the API thread (HostTier::take_frame
      // waits for its event) and drains the prefetch pipeline (50% pinned,
      // read_ahead 13: 9 GB/s). So leave the in-flight layers and as many
      // again untouched; a few layers of lead cover the read-in latency, and
      // every frame not needed for them stays resident (below): at 50%
      // pinned a cap of 6 layers gave 0.70-0.74 of the link, 4 or 2 gave 0.86
      // (profiles/r2t_tier_micro.jsonl).
      long long per_layer = 0;
      for (const Member& m : members) per_layer += m.nblk;
      const long long fit = per_layer > 0 ? cfg.pinned_frames / per_layer : L;
      constexpr long long kRaSlack = 2, kRaMax = 4;
      read_ahead = static_cast<int>(
          std::clamp<long long>(fit - 2 * cfg.pipeline_depth - kRaSlack, 0, std::min<long long>(L, kRaMax)));
      // the rest of the frames stay resident across iterations (HostTier::
      // set_sticky_budget): the staged layers, the one being fetched, the
      // ones in flight and one more cycle through the LRU frames
      tier.set_sticky_budget(cfg.pinned_frames - (read_ahead + cfg.pipeline_depth + 2) * per_layer);
      staged.assign(L, 0);
      staged_slots.assign(L, {});
      for (int l = 0; l < std::min(read_ahead + cfg.pipeline_depth, L); ++l) stage_layer(l);
    }
    for (int l = 0; l < std::min(cfg.pipeline_depth, L); ++l) issue_fetch(l);
  }

  // ---- v2: persistent warps, TMA bulk ring (decode_attn.cuh) ------------------
  // Chunk size: the largest power of two <= 32 that still deals every warp of
  // the persistent grid >= 8 units (load balance on ragged batches).
  // The tensor-core kernel deals units to CTAs instead of warps and works in
  // 128-token tiles: chunks of up to 16 tiles, never below one tile.
  void plan_chunks() {
    const bool tc_path = tc_decode();
    const long long workers = static_cast<long long>(sms) * (tc_path ? 1 : 12);
    const long long block_heads = static_cast<long long>(total_blocks) * Hl;
    const int tile_blocks = 128 / bs;
    int cb = tc_path ? 16 * tile_blocks : 32;
    const int cb_min = tc_path ? tile_blocks : 1;
    // units per worker before halving the chunk: the tensor-core kernel's
    // per-unit epilogue favours fewer, longer units (measured: 4 -> 85%, 8 ->
    // 81% on the 70B TP8 shard; flat on 8B; 2 and 1 within noise of 4,
    // profiles/r2ae_tc_units.jsonl), the CUDA-core one balances at 8
    // (profiles/r1y_decode_micro.jsonl).
    const long long per_worker = tc_path ? 4 : 8;
    while (cb > cb_min && block_heads / cb < per_worker * workers) cb >>= 1;
    std::vector<AttnChunk> ch;
    auto* aseq = reinterpret_cast<AttnSeq*>(ring.reserve(std::max<std::size_t>(members.size(), 1) * sizeof(AttnSeq)));
    for (std::size_t i = 0; i < members.size(); ++i) {
      const Member& m = members[i];
      aseq[i] = {m.blk_off, m.kv_len, static_cast<int>(ch.size()), (m.nblk + cb - 1) / cb};
      for (int b0 = 0; b0 < m.nblk; b0 += cb) ch.push_back({static_cast<int>(i), b0, std::min(cb, m.nblk - b0), 0});
    }
    LKV_CUDA(cudaMemcpyAsync(d_aseqs, aseq, std::max<std::size_t>(members.size(), 1) * sizeof(AttnSeq),
                             cudaMemcpyHostToDevice, cs));
    ring.commit(cs);
    n_chunks = static_cast<int>(ch.size());
    const long long units = static_cast<long long>(n_chunks) * Hl;
    if (units * G > part_cap) {  // grow the partial buffers (outside any kernel's lifetime)
      LKV_CUDA(cudaStreamSynchronize(cs));
      cudaFree(d_part_o);
      cudaFree(d_part_ml);
      part_cap = units * G * 2;
      LKV_CUDA(cudaMalloc(&d_part_o, part_cap * D * sizeof(float)));
      LKV_CUDA(cudaMalloc(&d_part_ml, part_cap * 2 * sizeof(float)));
    }
    if (static_cast<long long>(ch.size()) > chunk_cap) {
      LKV_CUDA(cudaStreamSynchronize(cs));
      cudaFree(d_chunks);
      chunk_cap = static_cast<long long>(ch.size()) * 2;
      LKV_CUDA(cudaMalloc(&d_chunks, chunk_cap * sizeof(AttnChunk)));
    }
    if (!ch.empty()) {
      auto* hc = reinterpret_cast<AttnChunk*>(ring.reserve(ch.size() * sizeof(AttnChunk)));
      std::memcpy(hc, ch.data(), ch.size() * sizeof(AttnChunk));
      LKV_CUDA(cudaMemcpyAsync(d_chunks, hc, ch.size() * sizeof(AttnChunk), cudaMemcpyHostToDevice, cs));
      ring.commit(cs);
    }
  }

  // Opt-in dynamic shared memory, once per kernel on this device (the
  // attribute is per device context, so it is tracked per lkv_device).
  std::unordered_set<const void*> smem_attr_done;
  void smem_attr(const void* fn, int bytes) {
    if (smem_attr_done.count(fn)) return;
    LKV_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    smem_attr_done.insert(fn);
  }

  // ---- v3: tcgen05 GQA tile (decode_gqa_tc.cuh) -------------------------------
  template <int GG, int BB>
  void launch_tc(int l, const void* q, float sl2) {
    constexpr int NS = 3;
    using K = GqaTc<GG, BB, NS>;
    auto fn = decode_gqa_tc_kernel<GG, BB, NS>;
    smem_attr(reinterpret_cast<const void*>(fn), K::kSmem);
    const int units = n_chunks * Hl;
    const int grid = std::max(1, std::min(sms, units));
    fn<<<grid, K::kThreads, K::kSmem, cs>>>(kvmap, Hl, d_snap + static_cast<long long>(l) * cfg.arena_slots,
                                            d_aseqs, d_chunks, units, static_cast<const __nv_bfloat16*>(q),
                                            d_part_o, d_part_ml, sl2, layer_stamps(l));
  }

  template <int GG>
  void launch_tc_bs(int l, const void* q, float sl2) {
    if (bs == 16) launch_tc<GG, 16>(l, q, sl2);
    else if (bs == 32) launch_tc<GG, 32>(l, q, sl2);
    else launch_tc<GG, 64>(l, q, sl2);
  }

  // G = 1: 12 warps x 2 stages per CTA (scripts/attn_micro.py, 7 x 16k, 7B:
  // 12x2 91% of HBM peak, 8x3 89%, 6x4 91%).
  template <int BB>
  void launch_v2(int l, const void* q, float sl2) {
    constexpr int W = 12, S = 2;
    using K = AttnV2<1, BB, W, S>;
    auto fn = decode_attn_v2_kernel<1, BB, W, S>;
    smem_attr(reinterpret_cast<const void*>(fn), K::kSmem);
    const int units = n_chunks * Hl;
    const int grid = std::max(1, std::min(sms, (units + W - 1) / W));
    fn<<<grid, K::kThreads, K::kSmem, cs>>>(dbuf, sb, Hl, d_snap + static_cast<long long>(l) * cfg.arena_slots,
                                            d_aseqs, d_chunks, units, static_cast<const __nv_bfloat16*>(q),
                                            d_part_o, d_part_ml, sl2, layer_stamps(l));
  }

  // f2: write each member's new token (position fetch_len) of layer l wherever
  // its slot lives. Destinations are resolved on the host from the manager's
  // table: the GPU slot, or the CPU slot's pinned frame plus its arena copy
  // (this step's attention reads the arena), or — offload in flight — the GPU
  // slot and the destination frame, after the D2H already carrying the block.
  void decode_append_layer(int l, const void* k, const void* v, cudaStream_t user) {
    if (!in_iteration || !append_mode)
      throw layersim::SimulationError("decode_append_layer outside decode_begin_append/end");
    check_layer(l);
    if (appended[l]) throw layersim::SimulationError("decode_append_layer: layer appended twice");
    const int st = l % cfg.pipeline_depth;
    const long long arena0 = cfg.gpu_slots + static_cast<long long>(st) * cfg.arena_slots;
    const int n = static_cast<int>(members.size());
    auto* dd = reinterpret_cast<AppendDesc*>(ring.reserve(std::max(n, 1) * sizeof(AppendDesc)));
    bool inflight = false;
    // host frames the token rows go to (tiered: pinned, read in first)
    std::vector<long long> hslots, hframes;
    for (int i = 0; i < n; ++i) {
      const RequestKv& r = kv->request(members[i].id);
      const auto& e = r.blocks[members[i].fetch_len / bs].layers[l];
      if (e.loc == Loc::Gpu && e.offload_in_flight) hslots.push_back(e.dest_slot);
      if (e.loc == Loc::Cpu) hslots.push_back(e.slot);
    }
    host_frames(hslots, true, &hframes);
    std::size_t hk = 0;
    for (int i = 0; i < n; ++i) {
      const Member& m = members[i];
      const RequestKv& r = kv->request(m.id);
      const int b = m.fetch_len / bs;
      const auto& e = r.blocks[b].layers[l];
      AppendDesc a{};
      a.tok = m.fetch_len % bs;
      if (e.loc == Loc::Gpu) {
        check_slot(e);
        a.dst[0] = dbuf + static_cast<long long>(e.slot) * sb;
        if (e.offload_in_flight) {
          if (static_cast<long long>(e.dest_slot) >= cfg.host_slots) throw CapacityError("append: dest frame");
          a.dst[1] = host_pool + hframes[hk++] * sb;
          inflight = true;
        }
      } else if (e.loc == Loc::Cpu) {
        check_slot(e);
        a.dst[0] = host_pool + hframes[hk++] * sb;
        a.dst[1] = dbuf + (arena0 + m.blk_off + b) * sb;
      } else {
        throw layersim::SimulationError("decode append: token slot has no location");
      }
      dd[i] = a;
    }
    join_in(user);
    LKV_CUDA(cudaStreamWaitEvent(cs, fetch_done[st], 0));  // the arena copy lands first
    if (inflight) {
      cudaEvent_t ev;
      ev_create(&ev);
      LKV_CUDA(cudaEventRecord(ev, d2h));
      LKV_CUDA(cudaStreamWaitEvent(cs, ev, 0));
      cudaEventDestroy(ev);
    }
    if (n > 0) {
      append_kv_kernel<<<n, 256, 0, cs>>>(dd, static_cast<const __nv_bfloat16*>(k),
                                          static_cast<const __nv_bfloat16*>(v), Hl, bs, D);
      LKV_CUDA(cudaGetLastError());
      dstats.kernel_launches += 1;
    }
    ring.commit(cs);
    host_done(hslots, cs, true);
    appended[l] = 1;
    join_out(user);
  }

  // Gather arguments of layer l's merge: a fresh epoch per decode_layer call
  // (every rank makes the same calls, so epochs agree across ranks).
  GatherArgs gather_args(int l) {
    GatherArgs ga{};
    if (!gather_on()) return ga;
    ++gather_epoch;
    layer_epoch[l] = gather_epoch;
    ga.bases = d_gather_bases;
    ga.n = cfg.tp_size;
    ga.rank = cfg.tp_rank;
    ga.hq_total = Hql * cfg.tp_size;
    ga.max_batch = cfg.max_batch;
    ga.parity = static_cast<int>(gather_epoch & 1u);
    ga.epoch = gather_epoch;
    ga.done = d_gather_done;
    return ga;
  }

  char* gather_buffer() {
    if (!d_gather) {
      gather_bytes = kGatherFlagWords * 4 + 2ull * gather_rows_per_parity() * D * 2;
      LKV_CUDA(cudaMalloc(&d_gather, gather_bytes));
      LKV_CUDA(cudaMemsetAsync(d_gather, 0, gather_bytes, cs));
      LKV_CUDA(cudaStreamSynchronize(cs));
    }
    return d_gather;
  }

  int gather_peers = 0;  // peers on other devices (P2P over NVLink)
  void gather_connect(const std::vector<char*>& bases) {
    if (static_cast<int>(bases.size()) != cfg.tp_size) throw std::invalid_argument("gather: need one base per rank");
    if (cfg.tp_size > kGatherFlagWords) throw std::invalid_argument("gather: too many ranks");
    if (bases[cfg.tp_rank] != gather_buffer()) throw std::invalid_argument("gather: own slot must be own buffer");
    // Peers' buffers on other GPUs: the merge kernel stores into them and the
    // wait kernel polls its own, so this device needs peer access to each
    // (IPC mappings enable it lazily; same-process peers need it explicitly).
    gather_peers = 0;
    for (int r = 0; r < cfg.tp_size; ++r) {
      if (r == cfg.tp_rank) continue;
      cudaPointerAttributes a{};
      LKV_CUDA(cudaPointerGetAttributes(&a, bases[r]));
      if (a.type != cudaMemoryTypeDevice) throw std::invalid_argument("gather: peer base is not device memory");
      if (a.device == cfg.device) continue;
      int can = 0;
      LKV_CUDA(cudaDeviceCanAccessPeer(&can, cfg.device, a.device));
      if (!can)
        throw CudaError("gather: device " + std::to_string(cfg.device) + " cannot access peer device " +
                        std::to_string(a.device) + " (no P2P path)");
      const cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else
        LKV_CUDA(e);
      ++gather_peers;
    }
    gather_bases = bases;
    if (!d_gather_bases) LKV_CUDA(cudaMalloc(&d_gather_bases, kGatherFlagWords * sizeof(char*)));
    if (!d_gather_done) LKV_CUDA(cudaMalloc(&d_gather_done, sizeof(unsigned)));
    LKV_CUDA(cudaMemcpy(d_gather_bases, bases.data(), bases.size() * sizeof(char*), cudaMemcpyHostToDevice));
    LKV_CUDA(cudaMemset(d_gather_done, 0, sizeof(unsigned)));
    layer_epoch.assign(L, 0);
  }

  // Merge v5 (4 warps: fits beside a persistent attention CTA) launched as a
  // programmatic dependent of the attention kernel.
  void launch_merge_v5(int n, void* out, int f32, GatherArgs ga) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(n, Hql);
    lc.blockDim = dim3(4 * 32);
    lc.dynamicSmemBytes = 0;
    lc.stream = cs;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    LKV_CUDA(cudaLaunchKernelEx(&lc, decode_merge_v5_kernel<4>, static_cast<const float*>(d_part_o),
                                static_cast<const float*>(d_part_ml), static_cast<const AttnSeq*>(d_aseqs), Hl, G,
                                out, f32, ga));
  }

  void decode_layer(int l, const void* q, void* out, float scale, int f32, cudaStream_t user) {
    if (!in_iteration) throw layersim::SimulationError("decode_layer outside decode_begin/end");
    check_layer(l);
    if (append_mode && !appended[l])
      throw layersim::SimulationError("decode_layer: append mode needs decode_append_layer first");
    const int st = l % cfg.pipeline_depth;
    join_in(user);
    LKV_CUDA(cudaStreamWaitEvent(cs, fetch_done[st], 0));
    const int n = static_cast<int>(members.size());
    if (timing) {
      LKV_CUDA(cudaEventRecord(t_attn0[l], cs));
    }
    if (n > 0) {
      const float sl2 = scale * 1.4426950408889634f;
      if (n_chunks > 0) {
        switch (G) {
          case 1:
            if (bs == 16) launch_v2<16>(l, q, sl2);
            else if (bs == 32) launch_v2<32>(l, q, sl2);
            else launch_v2<64>(l, q, sl2);
            break;
          case 2: launch_tc_bs<2>(l, q, sl2); break;
          case 4: launch_tc_bs<4>(l, q, sl2); break;
          default: launch_tc_bs<8>(l, q, sl2); break;
        }
        LKV_CUDA(cudaGetLastError());
      }
      // merge (members without KV get zero rows: no chunks, L = 0)
      launch_merge_v5(n, out, f32, gather_args(l));
      LKV_CUDA(cudaGetLastError());
      dstats.attn_launches += 1;
      dstats.kernel_launches += n_chunks > 0 ? 2 : 1;
    }
    if (n == 0 && gather_on()) {  // nothing to send, but peers still wait for this epoch
      const GatherArgs ga = gather_args(l);
      gather_flag_kernel<<<1, 1, 0, cs>>>(ga);
      LKV_CUDA(cudaGetLastError());
    }
    if (timing) {
      LKV_CUDA(cudaEventRecord(t_attnk[l], cs));  // attn_ms = the attention + merge pair
      LKV_CUDA(cudaEventRecord(t_attn1[l], cs));
    }
    LKV_CUDA(cudaEventRecord(attn_done[st], cs));
    attn_recorded[st] = 1;
    join_out(user);
    if (l + cfg.pipeline_depth < L) issue_fetch(l + cfg.pipeline_depth);
  }

  void decode_end() {
    if (!in_iteration) throw layersim::SimulationError("decode_end without decode_begin");
    in_iteration = false;
    if (tiered())  // layers staged but never fetched (an iteration cut short) give their frames back
      for (auto& s : staged_slots)
        if (!s.empty()) {
          tier.unstage(s.data(), static_cast<long long>(s.size()));
          s.clear();
        }
    if (timing) {
      LKV_CUDA(cudaStreamWaitEvent(cs, fetch_done[(L - 1) % cfg.pipeline_depth], 0));
      LKV_CUDA(cudaEventRecord(t_it1, cs));
    }
  }
};

// ============================================================================
#define LKV_TRY try {
#define LKV_CATCH                               \
  }                                             \
  catch (...) {                                 \
    return lkv::status_from_current_exception(); \
  }                                             \
  return LKV_OK;
#define LKV_REQUIRE(cond)                         \
  do {                                            \
    if (!(cond)) {                                \
      lkv::set_error("invalid argument: " #cond); \
      return LKV_ERR_INVALID;                     \
    }                                             \
  } while (0)

namespace lkv {
void device_bind_manager(lkv_device* d, KvManager& k) {
  if (k.n_layers() != d->L) throw std::invalid_argument("bind: layer count mismatch");
  if (k.tokens_per_block() != d->bs) throw std::invalid_argument("bind: tokens_per_block mismatch");
  if (!k.request_ids().empty()) throw std::invalid_argument("bind: manager already holds requests");
  d->kv = &k;
  d->free_full = true;
  k.set_observer(d);
}
// Completion event of an escalation job's last D2H copy (timing-capable);
// null once complete_offload consumed it.
cudaEvent_t device_job_event(lkv_device* d, std::int64_t job_id) {
  auto it = d->job_ev.find(job_id);
  return it == d->job_ev.end() ? nullptr : it->second;
}
}  // namespace lkv

extern "C" {

int lkv_device_create(const lkv_model_spec* m, int32_t tpb, const lkv_device_config* c,
                      lkv_device** out) {
  LKV_REQUIRE(m && c && out);
  lkv_device* d = new lkv_device();
  try {
    d->init(m, tpb, c);
  } catch (...) {
    const int st = lkv::status_from_current_exception();
    delete d;
    return st;
  }
  *out = d;
  return LKV_OK;
}

int lkv_device_numa_node(int32_t cuda_device, int32_t* node) {
  LKV_REQUIRE(node && cuda_device >= 0);
  *node = lkv::gpu_numa_node(cuda_device);
  return LKV_OK;
}

int lkv_device_destroy(lkv_device* d) {
  delete d;
  return LKV_OK;
}

int lkv_device_get_info(const lkv_device* d, lkv_device_info* o) {
  LKV_REQUIRE(d && o);
  o->slot_bytes = d->sb;
  o->kv_heads_local = d->Hl;
  o->q_heads_local = d->Hql;
  o->head_dim = d->D;
  o->tokens_per_block = d->bs;
  o->pool = d->dbuf;
  o->host_pool = d->host_pool;
  o->arena = d->dbuf + d->cfg.gpu_slots * d->sb;
  o->compute_stream = d->cs;
  o->d2h_stream = d->d2h;
  o->h2d_stream = d->h2d;
  o->numa_node = d->tiered() ? d->tier.numa_node() : d->host_mem.node();
  o->gather_peers = d->gather_peers;
  return LKV_OK;
}


int lkv_device_bind(lkv_device* d, lkv_kv_manager* kv) {
  LKV_REQUIRE(d && kv);
  LKV_TRY lkv::device_bind_manager(d, lkv::kv_impl(kv));
  LKV_CATCH
}

int lkv_device_synchronize(lkv_device* d) {
  LKV_REQUIRE(d);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  d->flush();
  LKV_CUDA(cudaStreamSynchronize(d->cs));
  LKV_CUDA(cudaStreamSynchronize(d->d2h));
  LKV_CUDA(cudaStreamSynchronize(d->h2d));
  LKV_CATCH
}

int lkv_prefill_layer(lkv_device* d, int64_t id, int32_t layer, const void* k, const void* v,
                      int64_t tokens, void* stream) {
  LKV_REQUIRE(d && k && v && tokens >= 0 && d->kv);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  d->prefill_layer(id, layer, k, v, tokens, static_cast<cudaStream_t>(stream));
  LKV_CATCH
}

int lkv_prefill_attention(lkv_device* d, const void* q, const void* k, const void* v, void* out, int64_t tokens,
                          float scale, int32_t out_dtype, void* stream) {
  LKV_REQUIRE(d && q && k && v && out && tokens >= 0);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  if (tokens == 0) return LKV_OK;
  if (tokens > 0x7FFFFF80ll) throw std::invalid_argument("prefill_attention: too many tokens");
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->cs;
  const uint64_t T = static_cast<uint64_t>(tokens), D = static_cast<uint64_t>(d->D);
  // fp16 copy of V in a device scratch (bf16 -> fp16 is exact in fp16's
  // normal range, saturating beyond it: the input contract in lkv.h)
  const std::size_t need = static_cast<std::size_t>(T) * d->Hl * D * 2;
  if (need > d->vh_cap) {
    LKV_CUDA(cudaDeviceSynchronize());
    cudaFree(d->d_vh);
    LKV_CUDA(cudaMalloc(&d->d_vh, need));
    d->vh_cap = need;
  }
  if (d->vh_used) LKV_CUDA(cudaStreamWaitEvent(s, d->vh_free, 0));  // previous user of the scratch
  const long long n8 = static_cast<long long>(need / 16);
  const int grid = static_cast<int>(std::min<long long>((n8 + 255) / 256, 8ll * d->sms));
  bf16_to_f16_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(v), static_cast<uint4*>(d->d_vh), n8);
  LKV_CUDA(cudaGetLastError());
  CUtensorMap qm, km, vm;
  if (!tc::make_map_3d(&qm, q, D, d->Hql, T, D * 2, D * 2 * d->Hql, 64, 1, 128, true) ||
      !tc::make_map_3d(&km, k, D, d->Hl, T, D * 2, D * 2 * d->Hl, 64, 1, 128, true) ||
      !tc::make_map_3d(&vm, d->d_vh, D, d->Hl, T, D * 2, D * 2 * d->Hl, 64, 1, 128, true,
                       CU_TENSOR_MAP_DATA_TYPE_FLOAT16))
    throw CudaError("prefill_attention: cuTensorMapEncodeTiled failed (pointers must be 16 B aligned)");
  const int nq_all = static_cast<int>((tokens + 127) / 128);
  // KV heads per dispatch chunk: as many as keep their K+V (T x 512 B per
  // KV head, bf16 K + fp16 V) within 16 MB of L2 (measured best of
  // 0 / 16 / 48 / 96 MB / all heads, profiles/r1ab_prefill_order.jsonl).
  constexpr long long kL2Budget = 16ll << 20;
  const long long kv_per_head = static_cast<long long>(tokens) * 512;
  const int chunk_kv = static_cast<int>(std::clamp<long long>(kL2Budget / std::max(kv_per_head, 1ll), 1, d->Hl));
  const int chunk_q = chunk_kv * d->G;
  const long long npairs_all = (nq_all + 1) / 2;
  auto fn2 = prefill_attn2_kernel;
  d->smem_attr(reinterpret_cast<const void*>(fn2), PrefillAttn2Smem::kBytes);
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(static_cast<unsigned>(npairs_all * d->Hql));
  lc.blockDim = dim3(kPrefillThreads);
  lc.dynamicSmemBytes = PrefillAttn2Smem::kBytes;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;  // dependent of bf16_to_f16_kernel
  lc.attrs = at;
  lc.numAttrs = 1;
  LKV_CUDA(cudaLaunchKernelEx(&lc, fn2, qm, km, vm, out, out_dtype == LKV_DTYPE_F32 ? 1 : 0,
                              static_cast<int>(tokens), d->Hql, d->G, scale * 1.4426950408889634f, chunk_q));
  LKV_CUDA(cudaGetLastError());
  LKV_CUDA(cudaEventRecord(d->vh_free, s));
  d->vh_used = true;
  LKV_CATCH
}

int lkv_device_job_done(lkv_device* d, int64_t job_id, int32_t* done) {
  LKV_REQUIRE(d && done);
  LKV_TRY auto it = d->job_ev.find(job_id);
  if (it == d->job_ev.end()) {
    *done = 1;
  } else {
    const cudaError_t e = cudaEventQuery(it->second);
    if (e != cudaSuccess && e != cudaErrorNotReady) LKV_CUDA(e);
    *done = e == cudaSuccess ? 1 : 0;
  }
  LKV_CATCH
}

int lkv_device_prefill_offload_done(lkv_device* d, int64_t id, int32_t* done) {
  LKV_REQUIRE(d && done);
  LKV_TRY auto it = d->prefill_ev.find(id);
  if (it == d->prefill_ev.end()) {
    *done = 1;
  } else {
    const cudaError_t e = cudaEventQuery(it->second);
    if (e != cudaSuccess && e != cudaErrorNotReady) LKV_CUDA(e);
    *done = e == cudaSuccess ? 1 : 0;
  }
  LKV_CATCH
}

int lkv_decode_begin(lkv_device* d, const int64_t* ids, int32_t n) {
  LKV_REQUIRE(d && d->kv && (ids || n == 0));
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  d->decode_begin(ids, n);
  LKV_CATCH
}

int lkv_decode_begin_append(lkv_device* d, const int64_t* ids, int32_t n) {
  LKV_REQUIRE(d && d->kv && (ids || n == 0));
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  d->decode_begin(ids, n, true);
  LKV_CATCH
}

int lkv_decode_append_layer(lkv_device* d, int32_t layer, const void* k_new, const void* v_new, void* stream) {
  LKV_REQUIRE(d && d->kv && k_new && v_new);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  d->decode_append_layer(layer, k_new, v_new, static_cast<cudaStream_t>(stream));
  LKV_CATCH
}

int lkv_decode_layer(lkv_device* d, int32_t layer, const void* q, void* out, float scale,
                     int32_t out_dtype, void* stream) {
  LKV_REQUIRE(d && d->kv && q && out);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  d->decode_layer(layer, q, out, scale, out_dtype == LKV_DTYPE_F32 ? 1 : 0, static_cast<cudaStream_t>(stream));
  LKV_CATCH
}

int lkv_device_gather_buffer(lkv_device* d, void** base, uint64_t* bytes) {
  LKV_REQUIRE(d && base && bytes);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  *base = d->gather_buffer();
  *bytes = d->gather_bytes;
  LKV_CATCH
}

static_assert(sizeof(cudaIpcMemHandle_t) == LKV_IPC_HANDLE_BYTES, "lkv.h LKV_IPC_HANDLE_BYTES");

int lkv_device_gather_ipc_handle(lkv_device* d, void* handle) {
  LKV_REQUIRE(d && handle);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  cudaIpcMemHandle_t h;
  LKV_CUDA(cudaIpcGetMemHandle(&h, d->gather_buffer()));
  std::memcpy(handle, &h, sizeof h);
  LKV_CATCH
}

int lkv_device_gather_connect_ipc(lkv_device* d, const void* handles, int32_t n) {
  LKV_REQUIRE(d && handles && n == d->cfg.tp_size);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  std::vector<char*> bases(n);
  for (int r = 0; r < n; ++r) {
    if (r == d->cfg.tp_rank) {
      bases[r] = d->gather_buffer();
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + r * sizeof h, sizeof h);
    void* p = nullptr;
    LKV_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    d->gather_opened.push_back(static_cast<char*>(p));
    bases[r] = static_cast<char*>(p);
  }
  d->gather_connect(bases);
  LKV_CATCH
}

int lkv_device_gather_connect(lkv_device* d, void* const* bases, int32_t n) {
  LKV_REQUIRE(d && bases && n == d->cfg.tp_size);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  std::vector<char*> b(n);
  for (int r = 0; r < n; ++r) b[r] = static_cast<char*>(bases[r]);
  d->gather_connect(b);
  LKV_CATCH
}

int lkv_decode_gather_wait(lkv_device* d, int32_t layer, void* stream) {
  LKV_REQUIRE(d && d->gather_on() && layer >= 0 && layer < d->L);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->cs;
  gather_wait_kernel<<<1, 32, 0, s>>>(reinterpret_cast<const unsigned*>(d->d_gather), d->cfg.tp_size,
                                      d->layer_epoch[layer]);
  LKV_CUDA(cudaGetLastError());
  LKV_CATCH
}

int lkv_decode_gathered(lkv_device* d, int32_t layer, void** rows) {
  LKV_REQUIRE(d && d->gather_on() && rows && layer >= 0 && layer < d->L);
  const long long parity = d->layer_epoch[layer] & 1u;
  *rows = d->d_gather + kGatherFlagWords * 4 + parity * d->gather_rows_per_parity() * d->D * 2;
  return LKV_OK;
}

int lkv_decode_end(lkv_device* d) {
  LKV_REQUIRE(d);
  LKV_TRY d->decode_end();
  LKV_CATCH
}

int lkv_device_set_timing(lkv_device* d, int32_t on) {
  LKV_REQUIRE(d);
  d->timing = on != 0;
  return LKV_OK;
}

int lkv_decode_last_stats(const lkv_device* dc, lkv_decode_stats* out) {
  LKV_REQUIRE(dc && out);
  lkv_device* d = const_cast<lkv_device*>(dc);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  *out = d->dstats;
  if (d->timing && !d->in_iteration) {
    LKV_CUDA(cudaEventSynchronize(d->t_it1));
    float ms = 0.f;
    double attn = 0.0, merge = 0.0;
    for (int l = 0; l < d->L; ++l) {
      if (cudaEventElapsedTime(&ms, d->t_attn0[l], d->t_attnk[l]) == cudaSuccess) attn += ms;
      if (cudaEventElapsedTime(&ms, d->t_attnk[l], d->t_attn1[l]) == cudaSuccess) merge += ms;
    }
    cudaGetLastError();
    out->attn_ms = attn;
    out->merge_ms = merge;
    if (d->d_stamps) {  // attention kernels' own span (%globaltimer), beside the event-timed interval
      std::vector<unsigned long long> st(static_cast<std::size_t>(d->L) * 2);
      LKV_CUDA(cudaMemcpy(st.data(), d->d_stamps, st.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      double k = 0.0;
      for (int l = 0; l < d->L; ++l) {
        const unsigned long long t0 = ~st[2 * l], t1 = st[2 * l + 1];
        if (st[2 * l] != 0ull && t1 > t0) k += static_cast<double>(t1 - t0) * 1e-6;
      }
      out->kernel_ms = k;
    }
    if (d->h2d_started && cudaEventElapsedTime(&ms, d->t_h2d0, d->t_h2d1) == cudaSuccess)
      out->h2d_span_ms = ms;
    cudaGetLastError();
    double busy = 0.0;
    for (int l = 0; l < d->L; ++l)
      if (d->fetched[l] && cudaEventElapsedTime(&ms, d->t_f0[l], d->t_f1[l]) == cudaSuccess) busy += ms;
    cudaGetLastError();
    out->h2d_ms = busy;
    if (cudaEventElapsedTime(&ms, d->t_it0, d->t_it1) == cudaSuccess) out->iteration_ms = ms;
    cudaGetLastError();
  }
  LKV_CATCH
}

int lkv_offload_last_stats(const lkv_device* dc, lkv_offload_stats* out, int32_t reset) {
  LKV_REQUIRE(dc && out);
  lkv_device* d = const_cast<lkv_device*>(dc);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  d->ostats.d2h_ms += lkv_device::drain_timed(d->d2h_timed);
  *out = d->ostats;
  if (reset) d->ostats = lkv_offload_stats{};
  LKV_CATCH
}

int lkv_fill_kv(lkv_device* d, void* k, void* v, int64_t tokens, int64_t token0, int32_t layer,
                uint64_t seed, void* stream) {
  LKV_REQUIRE(d && k && v && tokens >= 0 && token0 >= 0);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->cs;
  const long long total = tokens * d->Hl * d->D;
  if (total > 0) {
    const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, 8ll * d->sms));
    fill_kv_kernel<<<grid, 256, 0, s>>>(static_cast<__nv_bfloat16*>(k), static_cast<__nv_bfloat16*>(v),
                                        tokens, token0, layer, d->Hl, d->head0, d->D, seed);
    LKV_CUDA(cudaGetLastError());
  }
  LKV_CATCH
}

int lkv_fill_kv_tokens(lkv_device* d, void* k, void* v, const int64_t* positions, int32_t n, int32_t layer,
                       uint64_t seed, void* stream) {
  LKV_REQUIRE(d && k && v && (positions || n == 0) && n >= 0);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : d->cs;
  if (n > 0) {
    auto* pos = reinterpret_cast<long long*>(d->ring.reserve(n * sizeof(long long)));
    std::memcpy(pos, positions, n * sizeof(long long));
    const long long total = static_cast<long long>(n) * d->Hl * d->D;
    const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, 8ll * d->sms));
    fill_kv_tokens_kernel<<<grid, 256, 0, s>>>(static_cast<__nv_bfloat16*>(k), static_cast<__nv_bfloat16*>(v), pos,
                                               n, layer, d->Hl, d->head0, d->D, seed);
    LKV_CUDA(cudaGetLastError());
    d->ring.commit(s);
  }
  LKV_CATCH
}

static void request_pass(lkv_device* d, int64_t id, int64_t n_tokens, uint64_t seed, bool write,
                         int64_t* mism) {
  LKV_CUDA(cudaSetDevice(d->cfg.device));
  d->flush();
  const RequestKv& r = d->kv->request(id);
  const int row = d->row_for(id);
  const long long nb = std::min<long long>(static_cast<long long>(r.blocks.size()),
                                           (n_tokens + d->bs - 1) / d->bs);
  if (!write) LKV_CUDA(cudaMemsetAsync(d->d_counter, 0, sizeof(unsigned long long), d->cs));
  // Host frames may still be landing from D2H copies.
  LKV_CUDA(cudaStreamSynchronize(d->d2h));
  // Tiered: one layer at a time, its CPU slots pinned (read in) and their
  // frames published to the kernel through d_xlat.
  const int passes = d->tiered() ? d->L : 1;
  for (int p = 0; p < passes && nb > 0; ++p) {
    std::vector<long long> slots, frames;
    if (d->tiered()) {
      for (long long b = 0; b < nb; ++b) {
        const auto& e = r.blocks[b].layers[p];
        if (e.loc == Loc::Cpu) slots.push_back(e.slot);
      }
      d->host_frames(slots, true, &frames);
      if (!slots.empty()) {
        auto* up = reinterpret_cast<TableUpdate*>(d->ring.reserve(slots.size() * sizeof(TableUpdate)));
        for (std::size_t i = 0; i < slots.size(); ++i) up[i] = {slots[i], static_cast<int>(frames[i]), 0};
        table_apply_kernel<<<1, 256, 0, d->cs>>>(up, static_cast<int>(slots.size()), d->d_xlat, FreeSync{});
        LKV_CUDA(cudaGetLastError());
        d->ring.commit(d->cs);
      }
    }
    const int layer0 = d->tiered() ? p : 0;
    dim3 grid(static_cast<unsigned>(nb), d->tiered() ? 1 : d->L);
    const int* xl = d->tiered() ? d->d_xlat : nullptr;
    if (write)
      request_kv_kernel<true><<<grid, 256, 0, d->cs>>>(d->d_table + d->tindex(row, 0, 0), d->cfg.max_blocks,
                                                       layer0, n_tokens, d->dbuf, d->host_pool, xl, d->sb, d->Hl,
                                                       d->head0, d->bs, d->D, seed, d->d_counter);
    else
      request_kv_kernel<false><<<grid, 256, 0, d->cs>>>(d->d_table + d->tindex(row, 0, 0), d->cfg.max_blocks,
                                                        layer0, n_tokens, d->dbuf, d->host_pool, xl, d->sb, d->Hl,
                                                        d->head0, d->bs, d->D, seed, d->d_counter);
    LKV_CUDA(cudaGetLastError());
    d->host_done(slots, d->cs, write);
  }
  if (!write) {
    unsigned long long h = 0;
    LKV_CUDA(cudaMemcpyAsync(&h, d->d_counter, sizeof h, cudaMemcpyDeviceToHost, d->cs));
    LKV_CUDA(cudaStreamSynchronize(d->cs));
    *mism = static_cast<int64_t>(h);
  } else {
    LKV_CUDA(cudaStreamSynchronize(d->cs));
  }
}

int lkv_device_free_stack(lkv_device* d, int32_t which, uint32_t* out, int64_t cap, int64_t* size) {
  LKV_REQUIRE(d && (which == 0 || which == 1) && size && (out || cap == 0));
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  d->flush();
  long long hdr[6];
  LKV_CUDA(cudaMemcpyAsync(hdr, d->d_free_hdr, sizeof hdr, cudaMemcpyDeviceToHost, d->cs));
  LKV_CUDA(cudaStreamSynchronize(d->cs));
  const long long total = hdr[3 * which], fresh = hdr[3 * which + 1], pushed = hdr[3 * which + 2];
  *size = (total - fresh) + pushed;
  if (cap >= *size) {
    for (long long i = 0; i < total - fresh; ++i) out[i] = static_cast<uint32_t>(total - 1 - i);
    if (pushed > 0) {
      LKV_CUDA(cudaMemcpyAsync(out + (total - fresh), which == 0 ? d->d_free_gpu : d->d_free_cpu,
                               pushed * sizeof(unsigned), cudaMemcpyDeviceToHost, d->cs));
      LKV_CUDA(cudaStreamSynchronize(d->cs));
    }
  }
  LKV_CATCH
}

int lkv_device_read_host_slot(lkv_device* d, int64_t slot, void* dst) {
  LKV_REQUIRE(d && dst && slot >= 0 && slot < d->cfg.host_slots);
  LKV_TRY LKV_CUDA(cudaSetDevice(d->cfg.device));
  LKV_CUDA(cudaStreamSynchronize(d->d2h));
  LKV_CUDA(cudaStreamSynchronize(d->cs));
  if (d->tiered())
    d->tier.read_slot(slot, dst);
  else
    std::memcpy(dst, d->host_pool + slot * d->sb, static_cast<std::size_t>(d->sb));
  LKV_CATCH
}

int lkv_device_host_tier_stats(const lkv_device* d, lkv_host_tier_stats* o) {
  LKV_REQUIRE(d && o);
  std::memset(o, 0, sizeof *o);
  if (d->tier.enabled()) {
    const auto t = d->tier.stats();
    o->pinned_frames = d->tier.frames();
    o->read_in_frames = t.read_in_frames;
    o->write_back_frames = t.write_back_frames;
    o->evictions = t.evictions;
    o->hits = t.hits;
    o->misses = t.misses;
    o->staged = t.staged;
    o->pin_waits = t.pin_waits;
    o->read_ahead = d->read_ahead;
    o->resident_frames = d->tier.sticky_frames();
    o->copy_threads = d->tier.copy_threads();
  }
  return LKV_OK;
}

int lkv_verify_request(lkv_device* d, int64_t id, int64_t n_tokens, uint64_t seed,
                       int64_t* mismatches) {
  LKV_REQUIRE(d && d->kv && mismatches);
  LKV_TRY request_pass(d, id, n_tokens, seed, false, mismatches);
  LKV_CATCH
}

int lkv_fill_request(lkv_device* d, int64_t id, int64_t n_tokens, uint64_t seed) {
  LKV_REQUIRE(d && d->kv);
  LKV_TRY request_pass(d, id, n_tokens, seed, true, nullptr);
  LKV_CATCH
}

}  // extern "C"

#if LKV_PREFILL_TRACE
// Diagnostic builds only (scripts/build_variant.sh ... -DLKV_PREFILL_TRACE=1).
extern "C" __attribute__((visibility("default"))) int lkv_debug_prefill_trace(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, lkv::g_pf_trace, sizeof(unsigned long long) * std::min(n, 4096)) == cudaSuccess
             ? 0
             : -1;
}
extern "C" __attribute__((visibility("default"))) int lkv_debug_prefill_cta(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, lkv::g_pf_cta, sizeof(unsigned long long) * std::min(n, 3 * 4096)) == cudaSuccess
             ? 0
             : -1;
}
#endif
