// Two-tier host memory for CPU slots ("a
// CPU thread handles the transfer of KV cache from pinned memory to pageable
// memory").
//
// The reference sizes the CPU pool at cpu_pool_multiple x the GPU pool
// (kv_manager.hpp:24; 904,344 slots = 237 GB for config 2), far more than a
// host can pin. Tiered mode keeps every CPU slot's home in pageable memory
// (one MAP_NORESERVE mapping: pages exist only once written) and a bounded
// set of pinned, device-mapped frames as the DMA-facing tier:
//   - a D2H (prefill pack, escalation) or an in-kernel write (decode append)
//     lands in the slot's pinned frame; the frame is dirty until the cleaner
//     thread copies it home after the GPU work's event completes;
//   - an H2D prefetch or an in-kernel read needs the slot resident: a
//     missing slot is read in from its home into a frame by a persistent
//     pool of copy workers. stage() starts those read-ins without waiting
//     (the decode path stages layers several ahead of their DMA), pin()
//     waits only for the ones still running;
//   - a frame is reused least-recently-used first, never before its last
//     GPU use completed, never while locked (pinned or staged), being read
//     in or written home, and never while dirty (written back first);
//   - slots the manager frees are forgotten (no write-back).
// Homes and frames sit on the GPU's NUMA node. One mutex guards the frame
// table; the API thread, the cleaner and the copy workers take it briefly.
#pragma once

#include <cuda_runtime.h>
#include <emmintrin.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "host_mem.hpp"

namespace lkv {

struct HostTierStats {
  long long read_in_frames = 0, write_back_frames = 0, evictions = 0, hits = 0, misses = 0;
  long long staged = 0;      // slots staged ahead of their pin()
  long long pin_waits = 0;   // pin() calls that waited for a read-in still running
};

class HostTier {
 public:
  HostTier() = default;
  HostTier(const HostTier&) = delete;
  HostTier& operator=(const HostTier&) = delete;
  ~HostTier() { destroy(); }

  // slots: addressable CPU slots (pageable homes); frames: pinned frames.
  void init(int device, long long slots, long long frames, long long frame_bytes, int copy_threads, int numa_node) {
    device_ = device;
    S_ = slots;
    F_ = frames;
    sb_ = frame_bytes;
    void* p = mmap(nullptr, static_cast<std::size_t>(S_ * sb_), PROT_READ | PROT_WRITE,
                   MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (p == MAP_FAILED) throw std::runtime_error("host tier: mmap of the pageable homes failed");
    home_ = static_cast<char*>(p);
    // 2 MiB pages where the kernel allows them (THP "madvise" or "always"):
    // a 256 KiB frame copy touches 64 base pages otherwise.
    madvise(home_, static_cast<std::size_t>(S_ * sb_), MADV_HUGEPAGE);
    if (numa_node >= 0 && numa_node < 128) {  // homes follow the frames (pages are placed at first write)
      unsigned long mask[2] = {0ul, 0ul};
      mask[numa_node / 64] = 1ul << (numa_node % 64);
      syscall(SYS_mbind, home_, static_cast<std::size_t>(S_ * sb_), 1l /* MPOL_PREFERRED */, mask, 129ul, 0u);
    }
    threads_ = std::max(1, copy_threads);
    pinned_mem_.allocate(static_cast<std::size_t>(F_ * sb_), numa_node, threads_);
    pinned_ = pinned_mem_.data();
    slot_frame_.assign(static_cast<std::size_t>(S_), -1);
    slot_valid_.assign(static_cast<std::size_t>(S_), 0);
    frames_.resize(static_cast<std::size_t>(F_));
    // popped from the back: ascending frames, so a batch of misses gets a
    // contiguous run and its DMA coalesces into one copy
    for (long long f = F_ - 1; f >= 0; --f) free_.push_back(static_cast<int>(f));
    stop_ = false;
    for (int i = 0; i < threads_; ++i) workers_.emplace_back([this] { work_loop(); });
    cleaner_ = std::thread([this] { clean_loop(); });
  }

  void destroy() {
    if (cleaner_.joinable() || !workers_.empty()) {
      {
        std::lock_guard<std::mutex> g(mu_);
        stop_ = true;
      }
      {
        std::lock_guard<std::mutex> g(qmu_);
        qstop_ = true;
      }
      cv_.notify_all();
      qcv_.notify_all();
      if (cleaner_.joinable()) cleaner_.join();
      for (auto& t : workers_) t.join();
      workers_.clear();
    }
    frames_.clear();
    pinned_mem_.release();
    pinned_ = nullptr;
    if (home_) munmap(home_, static_cast<std::size_t>(S_ * sb_));
    home_ = nullptr;
  }

  bool enabled() const { return pinned_ != nullptr; }
  char* pinned() const { return pinned_; }
  long long frames() const { return F_; }
  int numa_node() const { return pinned_mem_.node(); }
  int copy_threads() const { return threads_; }
  HostTierStats stats() const {
    std::lock_guard<std::mutex> g(mu_);
    return st_;
  }

  // Up to `n` frames stay resident outside the LRU order: the next slots that
  // take a frame keep it until the manager frees them. A decode iteration
  // re-reads every CPU-resident slot in a fixed cyclic order, the access
  // pattern on which LRU always evicts the slot needed next (0% hits); a
  // fixed resident subset is the optimal policy there (hits = n / slots).
  // The caller leaves enough LRU frames for the layers in flight and staged.
  void set_sticky_budget(long long n) {
    std::lock_guard<std::mutex> g(mu_);
    sticky_budget_ = std::max(0ll, std::min(n, F_));
    while (sticky_count_ > sticky_budget_) {  // shrink: the oldest become ordinary LRU frames
      const int f = sticky_.front();
      sticky_.pop_front();
      Frame& fr = frames_[static_cast<std::size_t>(f)];
      fr.sticky = false;
      --sticky_count_;
      lru_.push_front(f);
      fr.pos = lru_.begin();
      fr.in_lru = true;
    }
  }
  long long sticky_frames() const {
    std::lock_guard<std::mutex> g(mu_);
    return sticky_count_;
  }

  // Read-ahead: make `slots` resident, starting the read-in of missing ones
  // on the copy workers without waiting for them. Every slot keeps one stage
  // lock (no eviction) until a pin() consumes it or unstage() drops it.
  void stage(const long long* slots, long long n) {
    std::vector<Job> jobs;
    {
      std::unique_lock<std::mutex> g(mu_);
      for (long long i = 0; i < n; ++i) {
        const int f = resident_or_take(g, slots[i], jobs);
        frames_[static_cast<std::size_t>(f)].stage_locks += 1;
      }
      st_.staged += n;
    }
    submit(jobs);
  }
  // Drops stage locks that no pin() consumed (an iteration that ended early).
  void unstage(const long long* slots, long long n) {
    std::lock_guard<std::mutex> g(mu_);
    for (long long i = 0; i < n; ++i) {
      const long long s = slots[i];
      if (s < 0 || s >= S_) continue;
      const int f = slot_frame_[static_cast<std::size_t>(s)];
      if (f >= 0 && frames_[static_cast<std::size_t>(f)].stage_locks > 0) frames_[static_cast<std::size_t>(f)].stage_locks -= 1;
    }
    cv_.notify_all();
  }

  // Frames for `n` slots, locked against eviction until the matching used()
  // call (a stage lock, if any, becomes that lock). read: the frame must hold
  // the slot's current bytes: waits for read-ins still running and reads in
  // the slots that were not staged.
  void pin(const long long* slots, long long n, bool read, long long* frames_out) {
    std::vector<Job> jobs;
    std::unique_lock<std::mutex> g(mu_);
    for (long long i = 0; i < n; ++i) {
      const long long s = slots[i];
      if (s < 0 || s >= S_) throw std::out_of_range("host tier: CPU slot " + std::to_string(s));
      const int f0 = slot_frame_[static_cast<std::size_t>(s)];
      const bool staged = f0 >= 0 && frames_[static_cast<std::size_t>(f0)].stage_locks > 0;  // counted by stage()
      const int f = resident_or_take(g, s, jobs, read, !staged);
      Frame& fr = frames_[static_cast<std::size_t>(f)];
      if (fr.stage_locks > 0) fr.stage_locks -= 1;
      fr.locks += 1;
      // a writer waits for a copy home of the frame's previous version to
      // finish (the generation count already kept such a copy from cleaning
      // the frame; this keeps the copy from reading bytes being replaced)
      if (!read && fr.cleaning) cv_.wait(g, [&] { return !fr.cleaning; });
      frames_out[i] = f;
    }
    g.unlock();
    submit(jobs);
    // a staged read-in still running must land before the caller reads the
    // frame, or before a GPU write replaces it (else it would overwrite it)
    g.lock();
    long long i0 = 0;  // frames before i0 have landed (resumes after each wake-up)
    auto filling = [&] {
      while (i0 < n && !frames_[static_cast<std::size_t>(frames_out[i0])].filling) ++i0;
      return i0 < n;
    };
    if (filling()) {
      ++st_.pin_waits;
      cv_.wait(g, [&] { return !filling(); });
    }
  }

  // The pinned frames of `slots` are used by GPU work that completes at `ev`
  // (an event recorded after that work); write: the GPU writes them.
  void used(const long long* slots, long long n, cudaEvent_t ev, bool write) {
    auto ticket = std::make_shared<Ticket>(ev);
    std::lock_guard<std::mutex> g(mu_);
    for (long long i = 0; i < n; ++i) {
      const int f = slot_frame_[static_cast<std::size_t>(slots[i])];
      if (f < 0) throw std::logic_error("host tier: used() on a slot that is not resident");
      Frame& fr = frames_[static_cast<std::size_t>(f)];
      fr.last = ticket;
      if (write) {
        if (!fr.dirty) dirty_q_.push_back(f);
        fr.dirty = true;
        fr.gen += 1;  // a copy home that started before this write does not clean it
        slot_valid_[static_cast<std::size_t>(slots[i])] = 1;
      }
      if (fr.locks > 0) fr.locks -= 1;
    }
    cv_.notify_all();
  }

  // The manager freed these slots: drop their bytes (no write-back).
  void forget(const long long* slots, long long n) {
    std::unique_lock<std::mutex> g(mu_);
    for (long long i = 0; i < n; ++i) {
      const long long s = slots[i];
      if (s < 0 || s >= S_) continue;
      slot_valid_[static_cast<std::size_t>(s)] = 0;
      const int f = slot_frame_[static_cast<std::size_t>(s)];
      if (f < 0) continue;
      Frame& fr = frames_[static_cast<std::size_t>(f)];
      // a copy of now-dead bytes (home or in) finishes first
      cv_.wait(g, [&] { return !fr.cleaning && !fr.filling; });
      if (slot_frame_[static_cast<std::size_t>(s)] != f) continue;
      fr.dirty = false;
      fr.stage_locks = 0;
      release_frame(f);
    }
    cv_.notify_all();
  }

  // Copy one slot's current bytes (resident or home) to `dst` (tests).
  void read_slot(long long s, void* dst) {
    std::unique_lock<std::mutex> g(mu_);
    const int f = slot_frame_[static_cast<std::size_t>(s)];
    if (f >= 0) {
      Frame& fr = frames_[static_cast<std::size_t>(f)];
      cv_.wait(g, [&] { return !fr.filling; });
      auto t = fr.last;
      g.unlock();
      if (t) cudaEventSynchronize(t->ev);
      std::memcpy(dst, pinned_ + f * sb_, static_cast<std::size_t>(sb_));
    } else {
      std::memcpy(dst, home_ + s * sb_, static_cast<std::size_t>(sb_));
    }
  }

 private:
  struct Ticket {
    // Owns the caller's event handle (recorded after the GPU work, never
    // re-recorded by it).
    explicit Ticket(cudaEvent_t src) : ev(src) {}
    ~Ticket() {
      if (ev) cudaEventDestroy(ev);
    }
    cudaEvent_t ev = nullptr;
  };
  struct Frame {
    long long slot = -1;
    bool dirty = false, cleaning = false, filling = false, in_lru = false, sticky = false;
    int locks = 0, stage_locks = 0;
    unsigned gen = 0;  // write generation
    std::shared_ptr<Ticket> last;
    std::list<int>::iterator pos;
  };
  struct Job {
    char* dst;
    const char* src;
    int frame;  // read-in: clears filling; -1: none
  };

  Job fill_job(int f) const {
    const Frame& fr = frames_[static_cast<std::size_t>(f)];
    return {pinned_ + f * sb_, home_ + fr.slot * sb_, f};
  }

  // The slot's frame, making it resident (a fresh frame) when needed; a
  // read-in job is appended to `jobs` when the slot holds bytes and `read`.
  // Called with mu_ held.
  int resident_or_take(std::unique_lock<std::mutex>& g, long long s, std::vector<Job>& jobs, bool read = true,
                       bool count = true) {
    if (s < 0 || s >= S_) throw std::out_of_range("host tier: CPU slot " + std::to_string(s));
    int f = slot_frame_[static_cast<std::size_t>(s)];
    if (f >= 0) {
      if (count) ++st_.hits;
      touch(f);
      return f;
    }
    if (count) ++st_.misses;
    f = take_frame(g, jobs);
    Frame& fr = frames_[static_cast<std::size_t>(f)];
    fr.slot = s;
    slot_frame_[static_cast<std::size_t>(s)] = f;
    if (sticky_count_ < sticky_budget_) {  // kept resident: never an eviction victim
      fr.sticky = true;
      ++sticky_count_;
      sticky_.push_back(f);
      fr.pos = std::prev(sticky_.end());
    } else {
      lru_.push_back(f);
      fr.pos = std::prev(lru_.end());
      fr.in_lru = true;
    }
    fr.filling = read && slot_valid_[static_cast<std::size_t>(s)];
    if (fr.filling) jobs.push_back(fill_job(f));
    return f;
  }

  void touch(int f) {
    Frame& fr = frames_[static_cast<std::size_t>(f)];
    if (fr.in_lru) lru_.splice(lru_.end(), lru_, fr.pos);
  }

  void release_frame(int f) {
    Frame& fr = frames_[static_cast<std::size_t>(f)];
    if (fr.slot >= 0) slot_frame_[static_cast<std::size_t>(fr.slot)] = -1;
    fr.slot = -1;
    if (fr.in_lru) {
      lru_.erase(fr.pos);
      fr.in_lru = false;
    } else if (fr.sticky) {
      sticky_.erase(fr.pos);
      fr.sticky = false;
      --sticky_count_;
    }
    free_.push_back(f);
  }

  static void wait_ticket(const std::shared_ptr<Ticket>& t) {
    if (t && t->ev) {
      const cudaError_t e = cudaEventSynchronize(t->ev);
      if (e != cudaSuccess) throw std::runtime_error(std::string("host tier: event: ") + cudaGetErrorString(e));
    }
  }

  static bool evictable(const Frame& fr) {
    return fr.locks == 0 && fr.stage_locks == 0 && !fr.cleaning && !fr.filling;
  }

  // A free frame, evicting the least recently used evictable one (its GPU
  // use completed; written home first when dirty). Called with mu_ held.
  // `pending`: read-ins the caller has not submitted yet; they are started
  // before this waits, since the frames they fill may be what it waits for.
  int take_frame(std::unique_lock<std::mutex>& g, std::vector<Job>& pending) {
    for (;;) {
      if (!free_.empty()) {  // a freed frame may still be read by an in-flight copy
        const int f = free_.back();
        free_.pop_back();
        Frame& fr = frames_[static_cast<std::size_t>(f)];
        auto t = std::move(fr.last);
        fr.dirty = false;
        fr.locks += 1;
        g.unlock();
        wait_ticket(t);
        g.lock();
        fr.locks -= 1;
        return f;
      }
      int victim = -1;
      for (int f : lru_)
        if (evictable(frames_[static_cast<std::size_t>(f)])) {
          victim = f;
          break;
        }
      if (victim < 0) {
        // the resident subset yields before anything waits or fails: the
        // budget is sized for decode iterations, and a prefill or escalation
        // in between may need more frames than the LRU part holds
        int keep = -1;
        for (int f : sticky_)
          if (evictable(frames_[static_cast<std::size_t>(f)])) {
            keep = f;
            break;
          }
        if (keep >= 0) {
          Frame& kf = frames_[static_cast<std::size_t>(keep)];
          sticky_.erase(kf.pos);
          kf.sticky = false;
          --sticky_count_;
          lru_.push_front(keep);
          kf.pos = lru_.begin();
          kf.in_lru = true;
          continue;  // it is the LRU victim now
        }
        if (!pending.empty()) {
          submit(pending);
          pending.clear();
        }
        bool busy = false;  // something that will make a frame evictable without this thread
        for (const std::list<int>* l : {&lru_, &sticky_})
          for (int f : *l) {
            const Frame& fr = frames_[static_cast<std::size_t>(f)];
            busy |= fr.cleaning || fr.filling;
          }
        if (!busy)
          throw std::length_error("host tier: every pinned frame is locked by work in flight (raise pinned_frames)");
        cv_.wait(g);
        continue;
      }
      Frame& fr = frames_[static_cast<std::size_t>(victim)];
      auto t = fr.last;
      const long long s = fr.slot;
      fr.locks += 1;  // hold while unlocked below
      g.unlock();
      wait_ticket(t);
      g.lock();
      fr.locks -= 1;
      if (!evictable(fr) || fr.slot != s) continue;  // re-locked meanwhile (a stage/pin of the same slot)
      if (fr.dirty) {  // the cleaner has not reached it: write it home here
        fr.cleaning = true;
        const unsigned gen = fr.gen;
        g.unlock();
        copy_frame(home_ + s * sb_, pinned_ + victim * sb_, static_cast<std::size_t>(sb_));
        g.lock();
        fr.cleaning = false;
        if (fr.gen == gen) fr.dirty = false;
        ++st_.write_back_frames;
        cv_.notify_all();
        if (fr.dirty || !evictable(fr) || fr.slot != s) continue;
      }
      ++st_.evictions;
      release_frame(victim);
      // loop: the frame is on the free list now
    }
  }

  // ---- copy workers (persistent; read-ins of stage() and pin())
  void submit(const std::vector<Job>& jobs) {
    if (jobs.empty()) return;
    {
      std::lock_guard<std::mutex> g(qmu_);
      for (const Job& j : jobs) q_.push_back(j);
    }
    if (jobs.size() == 1)
      qcv_.notify_one();
    else
      qcv_.notify_all();
  }

  void work_loop() {
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> g(qmu_);
        qcv_.wait(g, [&] { return qstop_ || !q_.empty(); });
        if (q_.empty()) return;  // stopping
        j = q_.front();
        q_.pop_front();
      }
      copy_frame(j.dst, j.src, static_cast<std::size_t>(sb_));
      if (j.frame >= 0) {
        std::lock_guard<std::mutex> g(mu_);
        frames_[static_cast<std::size_t>(j.frame)].filling = false;
        ++st_.read_in_frames;
      }
      cv_.notify_all();
    }
  }

  // The paper's CPU thread: copy dirty frames whose GPU writes completed to
  // their pageable homes, in the order they became dirty.
  void clean_loop() {
    cudaSetDevice(device_);
    std::unique_lock<std::mutex> g(mu_);
    while (!stop_) {
      int pick = -1;
      while (!dirty_q_.empty()) {
        const int f = dirty_q_.front();
        Frame& fr = frames_[static_cast<std::size_t>(f)];
        if (!fr.dirty || fr.cleaning) {  // cleaned or forgotten meanwhile (or being evicted)
          dirty_q_.pop_front();
          continue;
        }
        if (fr.locks == 0 && (!fr.last || !fr.last->ev || cudaEventQuery(fr.last->ev) == cudaSuccess)) {
          pick = f;
          dirty_q_.pop_front();
        }
        break;
      }
      if (pick < 0) {
        cv_.wait_for(g, std::chrono::milliseconds(1));
        continue;
      }
      Frame& fr = frames_[static_cast<std::size_t>(pick)];
      fr.cleaning = true;
      const long long s = fr.slot;
      const unsigned gen = fr.gen;
      g.unlock();
      copy_frame(home_ + s * sb_, pinned_ + pick * sb_, static_cast<std::size_t>(sb_));
      g.lock();
      fr.cleaning = false;
      if (fr.gen == gen) {
        fr.dirty = false;
      } else {
        dirty_q_.push_back(pick);  // written again meanwhile: stays dirty
      }
      ++st_.write_back_frames;
      cv_.notify_all();
    }
  }

  // Frame <-> home copy with non-temporal 16-byte stores: a 256 KiB frame
  // is never re-read by the CPU, so skipping the destination's
  // read-for-ownership saves a third of the host DRAM traffic the read-in
  // shares with the DMA reading the pinned frames
  // (profiles/r1y_tier_nt_micro.jsonl).
  static void copy_frame(char* dst, const char* src, std::size_t n) {
    if (((reinterpret_cast<std::uintptr_t>(dst) | reinterpret_cast<std::uintptr_t>(src) | n) & 63u) != 0u) {
      std::memcpy(dst, src, n);
      return;
    }
    for (std::size_t i = 0; i < n; i += 64) {
      const __m128i a = _mm_load_si128(reinterpret_cast<const __m128i*>(src + i));
      const __m128i b = _mm_load_si128(reinterpret_cast<const __m128i*>(src + i + 16));
      const __m128i c = _mm_load_si128(reinterpret_cast<const __m128i*>(src + i + 32));
      const __m128i d = _mm_load_si128(reinterpret_cast<const __m128i*>(src + i + 48));
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
    }
    _mm_sfence();
  }

  int device_ = 0;
  long long S_ = 0, F_ = 0, sb_ = 0;
  char* home_ = nullptr;
  PinnedHost pinned_mem_;
  char* pinned_ = nullptr;
  std::vector<int> slot_frame_;
  std::vector<std::uint8_t> slot_valid_;
  std::vector<Frame> frames_;
  std::vector<int> free_;
  std::list<int> lru_;
  std::list<int> sticky_;  // resident frames outside the LRU (set_sticky_budget)
  long long sticky_budget_ = 0, sticky_count_ = 0;
  std::deque<int> dirty_q_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
  std::thread cleaner_;
  bool stop_ = false;
  int threads_ = 8;
  HostTierStats st_;
  // copy workers
  std::vector<std::thread> workers_;
  std::deque<Job> q_;
  std::mutex qmu_;
  std::condition_variable qcv_;
  bool qstop_ = false;
};

}  // namespace lkv
