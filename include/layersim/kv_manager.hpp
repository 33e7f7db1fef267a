// Per-layer KV block table and GPU/CPU slot free lists — B200 drop-in for the
// reference allocator (proj/include/layersim/kv_manager.hpp:13-150).
//
// Public types and member functions are source compatible with the reference
// header, so the reference engine (proj/src/engine.cpp) compiles and links
// against this implementation unchanged. Observable state is bit-exact with
// the reference: every slot id handed out, the LIFO free-list order (including
// the re-ordering side effect of a rolled-back plan_offload), byte counts,
// exceptions and the dump_table text.
//
// What differs is the representation:
//   * free lists are O(1) to construct (implicit never-used range + explicit
//     LIFO stack), so 17.8 M-slot pools cost nothing until touched;
//   * every residency scan the reference does in O(blocks x layers)
//     (retained_layer_count, gpu_blocks_held, offload_reclaim,
//     plan_decode_fetch, select_offload_layers) is answered from per-layer
//     counters maintained incrementally, in O(layers);
//   * an optional KvObserver receives every table mutation; the B200 device
//     context (lkv::Device) implements it to mirror the table into HBM and to
//     drive the KV scatter / gather / offload / prefetch kernels.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <ostream>
#include <utility>
#include <vector>

#include "layersim/cost_model.hpp"
#include "layersim/errors.hpp"

namespace layersim {

struct BlockPools {
  std::int64_t gpu_blocks_total = 0;
  std::int64_t cpu_blocks_total = 0;
  int tokens_per_block = 16;
};

struct PoolSizing {
  std::int64_t max_input_tokens = 16384;
  int tokens_per_block = 16;
  double activation_layers_factor = 4.0;
  double cpu_pool_multiple = 8.0;
};

// Reference kv_manager.cpp:10-32. Throws ConfigError when nothing fits.
BlockPools pool_size_from_hardware(const ModelSpec& model, const HardwareSpec& hw,
                                   const PoolSizing& sizing);

struct PlacementPlan {
  std::vector<int> retained;   // ascending
  std::vector<int> offloaded;  // ascending complement
};

// retained = { floor((2j+1) L / 2x) }, reference kv_manager.cpp:34-50.
PlacementPlan layer_placement(int n_layers, int x);

enum class Loc : std::uint8_t { None, Gpu, Cpu };

struct SlotLoc {
  Loc loc = Loc::None;
  std::uint32_t slot = 0;
  bool offload_in_flight = false;
  std::uint32_t dest_slot = 0;
};

struct LogicalBlock {
  std::int64_t token_begin = 0;
  std::vector<SlotLoc> layers;
};

struct RequestKv {
  std::int64_t id = -1;
  std::int64_t cached_tokens = 0;
  std::vector<LogicalBlock> blocks;
  std::vector<Loc> layer_residency;
};

enum class OffloadMode { Half, Full };

struct OffloadJob {
  std::int64_t job_id = -1;
  std::int64_t request_id = -1;
  double bytes = 0.0;
  int layer_count = 0;
  std::int64_t gpu_blocks = 0;
};

struct FetchJob {
  int layer = 0;
  double bytes = 0.0;
};

// One (block, layer) entry moving GPU -> CPU in an escalation job, with the
// slots on both sides and the token-exact payload (reference
// kv_manager.cpp:251-257). Entries are in the reference's reservation order:
// selected layer ascending, then block ascending.
struct OffloadEntry {
  int block = 0;
  int layer = 0;
  std::uint32_t gpu_slot = 0;
  std::uint32_t cpu_slot = 0;
  std::int64_t filled_tokens = 0;
};

// Receives table mutations. All callbacks run synchronously on the caller's
// thread, after the table was updated unless stated otherwise.
class KvObserver {
 public:
  virtual ~KvObserver() = default;
  virtual void on_allocate(std::int64_t request_id, const RequestKv& kv) = 0;
  virtual void on_append(std::int64_t request_id, const RequestKv& kv) = 0;
  virtual void on_offload_planned(const OffloadJob& job,
                                  const std::vector<OffloadEntry>& entries) = 0;
  // Called BEFORE the job's GPU send buffers return to the free list, so the
  // device side can make sure the transfer out of them has drained.
  virtual void on_offload_complete(std::int64_t job_id, std::int64_t request_id,
                                   bool orphaned, const RequestKv* kv) = 0;
  // Called BEFORE the request's slots return to the free lists.
  virtual void on_release(std::int64_t request_id, const RequestKv& kv) = 0;
  // The manager is going away: drop every pointer into it.
  virtual void on_manager_destroyed() {}
};

class KvManager {
 public:
  KvManager(BlockPools pools, const ModelSpec& model);
  ~KvManager() {
    if (observer_) observer_->on_manager_destroyed();
  }
  // Copies are plain managers: a bound observer (the device mirror) stays with
  // the original, and a bound manager cannot be overwritten (its device table
  // would no longer describe it).
  KvManager(const KvManager& o)
      : pools_(o.pools_), n_layers_(o.n_layers_), kvb_(o.kvb_), gpu_(o.gpu_), cpu_(o.cpu_), tables_(o.tables_),
        pending_(o.pending_), next_job_id_(o.next_job_id_), observer_(nullptr) {}
  KvManager& operator=(const KvManager& o) {
    if (this != &o) {
      if (observer_) throw SimulationError("KvManager: assignment to a manager bound to a device observer");
      copy_from(o);
    }
    return *this;
  }

  int tokens_per_block() const { return pools_.tokens_per_block; }
  std::int64_t gpu_blocks_total() const { return pools_.gpu_blocks_total; }
  std::int64_t gpu_blocks_free() const { return gpu_.free_count(); }
  std::int64_t cpu_blocks_total() const { return pools_.cpu_blocks_total; }
  std::int64_t cpu_blocks_free() const { return cpu_.free_count(); }

  std::int64_t blocks_per_layer(std::int64_t tokens) const;
  std::int64_t request_wise_gpu_blocks(std::int64_t prompt_tokens) const;

  bool allocate_prefill(std::int64_t request_id, std::int64_t prompt_tokens, int x);

  bool has_request(std::int64_t request_id) const;
  const RequestKv& request(std::int64_t request_id) const;

  int retained_layer_count(std::int64_t request_id) const;
  std::int64_t gpu_blocks_held(std::int64_t request_id) const;
  std::int64_t gpu_row_cost(std::int64_t request_id) const;
  std::int64_t cpu_row_cost(std::int64_t request_id) const;
  std::int64_t offload_reclaim(std::int64_t request_id, OffloadMode mode) const;

  std::optional<OffloadJob> plan_offload(std::int64_t request_id, OffloadMode mode);
  void complete_offload(std::int64_t job_id);

  std::vector<FetchJob> plan_decode_fetch(std::int64_t request_id) const;

  bool needs_append(std::int64_t request_id) const;
  bool append_decode_block(std::int64_t request_id);
  void note_token(std::int64_t request_id);

  struct FreedCounts {
    std::int64_t gpu = 0;
    std::int64_t cpu = 0;
    std::int64_t deferred_gpu = 0;
  };
  FreedCounts release(std::int64_t request_id);

  void check_conservation() const;
  void dump_table(std::ostream& os) const;

  // ---- B200 additions (not in the reference API) ----
  int n_layers() const { return n_layers_; }
  std::int64_t kv_bytes_per_token_layer() const { return kvb_; }
  void set_observer(KvObserver* obs) { observer_ = obs; }
  // Entries of a pending escalation job (empty vector for unknown ids).
  const std::vector<OffloadEntry>& offload_entries(std::int64_t job_id) const;
  std::int64_t pending_offload_count() const { return static_cast<std::int64_t>(pending_.size()); }
  // Ids of live requests, ascending.
  std::vector<std::int64_t> request_ids() const;
  // Token-exact bytes of CPU-resident KV of layer `layer` (the per-layer
  // plan_decode_fetch value, 0 when nothing is on the CPU).
  std::int64_t cpu_layer_bytes(std::int64_t request_id, int layer) const;
  // Free-list journal for the device mirror. A LIFO stack
  // (kv_manager.cpp:52-74) is [total-1 ... next_fresh] + pushed[0..size):
  // between two takes, pops only shrink `pushed` to a low-water mark and
  // pushes append above it, so the change is (next_fresh, low, size,
  // pushed[low..size)). `full` restarts from low = 0.
  struct FreeListDelta {
    std::int64_t next_fresh = 0, low = 0, size = 0;
    const std::uint32_t* pushed = nullptr;  // the whole pushed stack; entries [low, size) changed
    bool changed = false;
  };
  FreeListDelta take_free_delta(bool gpu, bool full = false);
  // The stack itself: next_fresh and the pushed part (top = back).
  void free_stack(bool gpu, std::int64_t* next_fresh, std::vector<std::uint32_t>* pushed) const;

 private:
  // LIFO slot stack. The reference seeds its stack with total-1 ... 0 so the
  // first pop returns 0 (kv_manager.cpp:52-58). That stack always equals
  // [total-1 ... next_fresh_] followed by the explicitly pushed slots, so only
  // the pushed part is stored: pops take the explicit top when present, else
  // next_fresh_++.
  class FreeList {
   public:
    explicit FreeList(std::int64_t total);
    bool pop(std::uint32_t* slot);
    void push(std::uint32_t slot);  // throws SimulationError on a slot not held
    std::int64_t free_count() const {
      return static_cast<std::int64_t>(pushed_.size()) + (total_ - next_fresh_);
    }
    bool held(std::uint32_t slot) const;
    std::int64_t high_water() const { return next_fresh_; }
    FreeListDelta take_delta(bool full);
    const std::vector<std::uint32_t>& pushed() const { return pushed_; }

   private:
    std::int64_t total_;
    std::int64_t next_fresh_ = 0;
    std::vector<std::uint32_t> pushed_;
    std::vector<std::uint64_t> held_bits_;  // grows with next_fresh_
    // journal state of the device mirror: lowest pushed_.size() since the
    // last take_delta, and next_fresh_ / pushed_.size() at that take
    std::int64_t low_ = 0, fresh_taken_ = 0, size_taken_ = 0;
  };

  struct Table {
    RequestKv kv;
    std::vector<std::int32_t> gpu_live;   // per layer: loc==Gpu && !in_flight
    std::vector<std::int32_t> cpu_count;  // per layer: loc==Cpu
    std::int64_t gpu_held = 0;            // entries with loc==Gpu (incl. in flight)
    std::int64_t gpu_rows = 0;            // layer_residency == Gpu
    std::vector<std::int64_t> jobs;       // pending escalation ids, ascending
  };

  struct Pending {
    std::int64_t request_id = -1;
    std::vector<OffloadEntry> entries;
    std::vector<std::uint32_t> orphan_gpu;
    std::vector<std::uint32_t> orphan_cpu;
    bool orphaned = false;
  };

  Table& table(std::int64_t request_id);
  const Table& table(std::int64_t request_id) const;
  void select_layers(const Table& t, OffloadMode mode, std::vector<int>* out) const;
  std::int64_t filled(const RequestKv& kv, std::size_t block) const;

  void copy_from(const KvManager& o) {
    pools_ = o.pools_;
    n_layers_ = o.n_layers_;
    kvb_ = o.kvb_;
    gpu_ = o.gpu_;
    cpu_ = o.cpu_;
    tables_ = o.tables_;
    pending_ = o.pending_;
    next_job_id_ = o.next_job_id_;
    observer_ = nullptr;
  }

  BlockPools pools_;
  int n_layers_;
  std::int64_t kvb_;
  FreeList gpu_;
  FreeList cpu_;
  std::map<std::int64_t, Table> tables_;
  std::map<std::int64_t, Pending> pending_;
  std::int64_t next_job_id_ = 0;
  KvObserver* observer_ = nullptr;
};

}  // namespace layersim
