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
//     missing slot is read in from its home (parallel memcpy) into a frame
//     before the copy is enqueued;
//   - a frame is reused least-recently-used first, never before its last
//     GPU use completed, and never while dirty (written back first);
//   - slots the manager frees are forgotten (no write-back).
// Single writer (the device's API thread) + the cleaner thread, one mutex.
#pragma once

#include <cuda_runtime.h>
#include <emmintrin.h>
#include <sys/mman.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace lkv {

struct HostTierStats {
  long long read_in_frames = 0, write_back_frames = 0, evictions = 0, hits = 0, misses = 0;
};

class HostTier {
 public:
  HostTier() = default;
  HostTier(const HostTier&) = delete;
  HostTier& operator=(const HostTier&) = delete;
  ~HostTier() { destroy(); }

  // slots: addressable CPU slots (pageable homes); frames: pinned frames.
  void init(int device, long long slots, long long frames, long long frame_bytes, int copy_threads = 8) {
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
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&pinned_), static_cast<std::size_t>(F_ * sb_),
                                  cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) throw std::runtime_error(std::string("host tier: cudaHostAlloc: ") + cudaGetErrorString(e));
    slot_frame_.assign(static_cast<std::size_t>(S_), -1);
    slot_valid_.assign(static_cast<std::size_t>(S_), 0);
    frames_.resize(static_cast<std::size_t>(F_));
    // popped from the back: ascending frames, so a batch of misses gets a
    // contiguous run and its DMA coalesces into one copy
    for (long long f = F_ - 1; f >= 0; --f) free_.push_back(static_cast<int>(f));
    threads_ = std::max(1, copy_threads);
    stop_ = false;
    cleaner_ = std::thread([this] { clean_loop(); });
  }

  void destroy() {
    if (cleaner_.joinable()) {
      {
        std::lock_guard<std::mutex> g(mu_);
        stop_ = true;
      }
      cv_.notify_all();
      cleaner_.join();
    }
    frames_.clear();
    if (pinned_) cudaFreeHost(pinned_);
    pinned_ = nullptr;
    if (home_) munmap(home_, static_cast<std::size_t>(S_ * sb_));
    home_ = nullptr;
  }

  bool enabled() const { return pinned_ != nullptr; }
  char* pinned() const { return pinned_; }
  long long frames() const { return F_; }
  HostTierStats stats() const {
    std::lock_guard<std::mutex> g(mu_);
    return st_;
  }

  // Frames for `n` slots, locked against eviction until the matching used()
  // call. read: the frame must hold the slot's current bytes.
  void pin(const long long* slots, long long n, bool read, long long* frames_out) {
    std::unique_lock<std::mutex> g(mu_);
    std::vector<std::pair<long long, int>> fills;  // (slot, frame) to read in
    for (long long i = 0; i < n; ++i) {
      const long long s = slots[i];
      if (s < 0 || s >= S_) throw std::out_of_range("host tier: CPU slot " + std::to_string(s));
      int f = slot_frame_[static_cast<std::size_t>(s)];
      if (f >= 0) {
        ++st_.hits;
        touch(f);
      } else {
        ++st_.misses;
        f = take_frame(g);
        Frame& fr = frames_[static_cast<std::size_t>(f)];
        fr.slot = s;
        slot_frame_[static_cast<std::size_t>(s)] = f;
        lru_.push_back(f);
        fr.pos = std::prev(lru_.end());
        fr.in_lru = true;
        if (read && slot_valid_[static_cast<std::size_t>(s)]) fills.emplace_back(s, f);
      }
      frames_[static_cast<std::size_t>(f)].locks += 1;
      frames_out[i] = f;
    }
    g.unlock();
    if (!fills.empty()) {  // pageable homes -> pinned frames, in parallel
      copy_parallel(fills.size(), [&](std::size_t k) {
        copy_frame(pinned_ + fills[k].second * sb_, home_ + fills[k].first * sb_, static_cast<std::size_t>(sb_));
      });
      std::lock_guard<std::mutex> g2(mu_);
      st_.read_in_frames += static_cast<long long>(fills.size());
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
        fr.dirty = true;
        fr.gen += 1;  // a copy home that started before this write does not clean it
        slot_valid_[static_cast<std::size_t>(slots[i])] = 1;
      }
      if (fr.locks > 0) fr.locks -= 1;
    }
    if (write) cv_.notify_all();
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
      while (fr.cleaning) cv_.wait(g);  // the cleaner's copy of now-dead bytes finishes first
      if (slot_frame_[static_cast<std::size_t>(s)] != f) continue;
      fr.dirty = false;
      release_frame(f);
    }
  }

  // Copy one slot's current bytes (resident or home) to `dst` (tests).
  void read_slot(long long s, void* dst) {
    std::unique_lock<std::mutex> g(mu_);
    const int f = slot_frame_[static_cast<std::size_t>(s)];
    if (f >= 0) {
      auto t = frames_[static_cast<std::size_t>(f)].last;
      g.unlock();
      if (t) cudaEventSynchronize(t->ev);
      std::memcpy(dst, pinned_ + f * sb_, static_cast<std::size_t>(sb_));
    } else {
      std::memcpy(dst, home_ + s * sb_, static_cast<std::size_t>(sb_));
    }
  }

 private:
  struct Ticket {
    explicit Ticket(cudaEvent_t src) {
      // own a copy of the completion point: record-after is not available,
      // so the caller's event handle is kept and never re-recorded by it.
      ev = src;
    }
    ~Ticket() {
      if (ev) cudaEventDestroy(ev);
    }
    cudaEvent_t ev = nullptr;
  };
  struct Frame {
    long long slot = -1;
    bool dirty = false, cleaning = false, in_lru = false;
    int locks = 0;
    unsigned gen = 0;  // write generation
    std::shared_ptr<Ticket> last;
    std::list<int>::iterator pos;
  };

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
    }
    free_.push_back(f);
  }

  static void wait_ticket(const std::shared_ptr<Ticket>& t) {
    if (t && t->ev) {
      const cudaError_t e = cudaEventSynchronize(t->ev);
      if (e != cudaSuccess) throw std::runtime_error(std::string("host tier: event: ") + cudaGetErrorString(e));
    }
  }

  // A free frame, evicting the least recently used unlocked one (its GPU use
  // completed; written home first when dirty). Called with mu_ held.
  int take_frame(std::unique_lock<std::mutex>& g) {
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
      for (int f : lru_) {
        const Frame& fr = frames_[static_cast<std::size_t>(f)];
        if (fr.locks == 0 && !fr.cleaning) {
          victim = f;
          break;
        }
      }
      if (victim < 0) {
        bool any_cleaning = false;
        for (int f : lru_) any_cleaning |= frames_[static_cast<std::size_t>(f)].cleaning;
        if (!any_cleaning)
          throw std::length_error("host tier: every pinned frame is locked by the current batch (raise pinned_frames)");
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
      if (fr.dirty) {  // the cleaner has not reached it: write it home here
        fr.cleaning = true;
        g.unlock();
        copy_frame(home_ + s * sb_, pinned_ + victim * sb_, static_cast<std::size_t>(sb_));
        g.lock();
        fr.cleaning = false;
        fr.dirty = false;
        ++st_.write_back_frames;
      }
      ++st_.evictions;
      release_frame(victim);
      // loop: the frame is on the free list now
    }
  }

  // The paper's CPU thread: copy dirty frames whose GPU writes completed to
  // their pageable homes, oldest first.
  void clean_loop() {
    cudaSetDevice(device_);
    std::unique_lock<std::mutex> g(mu_);
    while (!stop_) {
      int pick = -1;
      for (int f : lru_) {
        Frame& fr = frames_[static_cast<std::size_t>(f)];
        if (fr.dirty && !fr.cleaning && fr.locks == 0 &&
            (!fr.last || !fr.last->ev || cudaEventQuery(fr.last->ev) == cudaSuccess)) {
          pick = f;
          break;
        }
      }
      if (pick < 0) {
        cv_.wait_for(g, std::chrono::milliseconds(2));
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
      if (fr.gen == gen) fr.dirty = false;  // else written again meanwhile: stays dirty
      ++st_.write_back_frames;
      cv_.notify_all();
    }
  }

  // Frame <-> home copy with non-temporal 16-byte stores: a 256 KiB frame
  // is never re-read by the CPU, so skipping the destination's
  // read-for-ownership saves a third of the host DRAM traffic the read-in
  // shares with the DMA reading the pinned frames.
  static void stream_copy(char* dst, const char* src, std::size_t n) {
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

  // Non-temporal stores: frames are not re-read by this CPU, so they skip
  // the cache (profiles/r1y_tier_nt_micro.jsonl).
  void copy_frame(char* dst, const char* src, std::size_t n) const { stream_copy(dst, src, n); }

  template <class Fn>
  void copy_parallel(std::size_t n, Fn&& fn) {
    const int t = static_cast<int>(std::min<std::size_t>(static_cast<std::size_t>(threads_), (n + 3) / 4));
    if (t <= 1) {
      for (std::size_t k = 0; k < n; ++k) fn(k);
      return;
    }
    std::atomic<std::size_t> next{0};
    std::vector<std::thread> pool;
    pool.reserve(static_cast<std::size_t>(t - 1));
    auto work = [&] {
      for (std::size_t k = next.fetch_add(1); k < n; k = next.fetch_add(1)) fn(k);
    };
    for (int i = 1; i < t; ++i) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
  }

  int device_ = 0;
  long long S_ = 0, F_ = 0, sb_ = 0;
  char* home_ = nullptr;
  char* pinned_ = nullptr;
  std::vector<int> slot_frame_;
  std::vector<std::uint8_t> slot_valid_;
  std::vector<Frame> frames_;
  std::vector<int> free_;
  std::list<int> lru_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
  std::thread cleaner_;
  bool stop_ = false;
  int threads_ = 8;
  HostTierStats st_;
};

}  // namespace lkv
