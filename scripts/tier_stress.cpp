// Concurrency stress of the two-tier host memory (csrc/host_tier.hpp) for
// the sanitizers (scripts/sanitize_host.sh): the real HostTier — API thread,
// copy workers, cleaner — against a simulated copy engine (one FIFO thread,
// like a CUDA stream) built on the host-only CUDA stub
// (scripts/cuda_stub/cuda_runtime.h). Not product code.
//
// The API thread issues, like lkv_device does: D2H-style writes (pin(read =
// false), the "engine" fills the frames with the slot's next version, then
// used(write)), H2D-style reads (optionally staged layers ahead, then
// pin(read = true); the engine checks every frame holds the slot's latest
// version), forgets (the manager freed the slots) and unstages. Any stale,
// torn or lost frame is counted as a mismatch; the run fails on any.
#include <cuda_runtime.h>

#include <cstdio>
#include <deque>
#include <functional>
#include <random>
#include <thread>
#include <string>
#include <vector>

#include "host_tier.hpp"

namespace {

constexpr long long kSlots = 3072, kFrames = 384, kSb = 4096;

struct Engine {  // the simulated copy engine: jobs run in submission order
  std::deque<std::function<void()>> q;
  std::mutex m;
  std::condition_variable cv;
  bool stop = false;
  std::thread th{[this] { run(); }};
  void run() {
    std::mt19937 rng(7);
    for (;;) {
      std::function<void()> f;
      {
        std::unique_lock<std::mutex> g(m);
        cv.wait(g, [&] { return stop || !q.empty(); });
        if (q.empty()) return;
        f = std::move(q.front());
        q.pop_front();
      }
      if (rng() % 4 == 0) std::this_thread::sleep_for(std::chrono::microseconds(rng() % 200));
      f();
    }
  }
  void submit(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> g(m);
      q.push_back(std::move(f));
    }
    cv.notify_one();
  }
  ~Engine() {
    {
      std::lock_guard<std::mutex> g(m);
      stop = true;
    }
    cv.notify_one();
    th.join();
  }
};

std::uint64_t word(long long slot, unsigned version, long long i) {
  return (static_cast<std::uint64_t>(slot) << 40) ^ (static_cast<std::uint64_t>(version) << 16) ^
         static_cast<std::uint64_t>(i);
}

}  // namespace

// A pin() wider than the pinned pool, over slots that hold bytes, must fail
// loudly: the read-ins it has not submitted yet fill the only frames it could
// wait for (the round-2 read-ahead rework deadlocked here instead).
int too_small() {
  int rc = 0;
  for (int staged = 0; staged < 2; ++staged) {
    auto* tier = new lkv::HostTier;  // leaked: its frames stay locked by the failed call
    tier->init(0, 64, 4, kSb, 2, -1);
    std::vector<long long> s(40), fr(40);
    for (int i = 0; i < 40; ++i) s[static_cast<std::size_t>(i)] = i;
    for (int i = 0; i < 40; i += 4) {  // give every slot bytes (written home through the tier)
      tier->pin(s.data() + i, 4, false, fr.data());
      cudaEvent_t ev = stub_event_new();
      stub_event_complete(ev);
      tier->used(s.data() + i, 4, ev, true);
    }
    try {
      if (staged)
        tier->stage(s.data(), 40);
      else
        tier->pin(s.data(), 40, true, fr.data());
      std::printf("too small (%s): no error\n", staged ? "stage" : "pin");
      rc = 1;
    } catch (const std::length_error& e) {
      std::printf("too small (%s): %s\n", staged ? "stage" : "pin", e.what());
    }
  }
  std::fflush(stdout);
  std::_Exit(rc);  // no orderly teardown of the leaked tiers
}

// The decode iteration's access pattern (lkv_device: stage read_ahead layers
// ahead, pin + DMA one layer, repeat every step): with a resident budget the
// slots of the first layers must hit from the second iteration on.
int cyclic(long long budget_layers) {
  const int L = 16, per_layer = 64, depth = 2, ra = 2;
  const long long slots = static_cast<long long>(L) * per_layer, frames = slots / 4;
  lkv::HostTier tier;
  tier.init(0, slots, frames, kSb, 4, -1);
  auto layer_slots = [&](int l) {
    std::vector<long long> v(per_layer);
    for (int i = 0; i < per_layer; ++i) v[static_cast<std::size_t>(i)] = static_cast<long long>(l) * per_layer + i;
    return v;
  };
  for (int l = 0; l < L; ++l) {  // every slot written once (the prefill offload)
    auto v = layer_slots(l);
    std::vector<long long> fr(v.size());
    tier.pin(v.data(), per_layer, false, fr.data());
    cudaEvent_t ev = stub_event_new();
    stub_event_complete(ev);
    tier.used(v.data(), per_layer, ev, true);
  }
  long long hits_last = 0;
  for (int it = 0; it < 4; ++it) {
    tier.set_sticky_budget(budget_layers * per_layer);
    const auto h0 = tier.stats().hits;
    std::vector<char> staged(L, 0);
    auto stage = [&](int l) {
      if (l >= L || staged[static_cast<std::size_t>(l)]) return;
      staged[static_cast<std::size_t>(l)] = 1;
      auto v = layer_slots(l);
      tier.stage(v.data(), per_layer);
    };
    for (int l = 0; l < std::min(L, ra + depth); ++l) stage(l);
    for (int l = 0; l < L; ++l) {
      auto v = layer_slots(l);
      std::vector<long long> fr(v.size());
      tier.pin(v.data(), per_layer, true, fr.data());
      cudaEvent_t ev = stub_event_new();
      stub_event_complete(ev);
      tier.used(v.data(), per_layer, ev, false);
      stage(l + ra);
    }
    hits_last = tier.stats().hits - h0;
    std::printf("cyclic: iteration %d, hits %lld of %lld, resident %lld\n", it, hits_last, slots, tier.sticky_frames());
  }
  return hits_last >= budget_layers * per_layer ? 0 : 1;
}

// A resident budget of nearly every frame must not starve a pin() wider
// than the LRU part (a prefill between decode iterations): resident frames
// yield, the pin succeeds.
int resident_yields() {
  lkv::HostTier tier;
  tier.init(0, 256, 64, kSb, 2, -1);
  tier.set_sticky_budget(60);
  std::vector<long long> s(64), fr(64);
  for (int i = 0; i < 64; ++i) s[static_cast<std::size_t>(i)] = i;  // fills all 64 frames, 60 resident
  tier.pin(s.data(), 64, false, fr.data());
  cudaEvent_t ev = stub_event_new();
  stub_event_complete(ev);
  tier.used(s.data(), 64, ev, true);
  std::vector<long long> t(48), ft(48);
  for (int i = 0; i < 48; ++i) t[static_cast<std::size_t>(i)] = 100 + i;  // 48 new slots at once
  try {
    tier.pin(t.data(), 48, false, ft.data());
  } catch (const std::exception& e) {
    std::printf("resident yields: failed: %s\n", e.what());
    return 1;
  }
  cudaEvent_t ev2 = stub_event_new();
  stub_event_complete(ev2);
  tier.used(t.data(), 48, ev2, true);
  std::printf("resident yields: ok, resident now %lld\n", tier.sticky_frames());
  tier.destroy();
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "small") return too_small();
  if (argc > 1 && std::string(argv[1]) == "yield") return resident_yields();
  if (argc > 2 && std::string(argv[1]) == "cyclic") return cyclic(std::atoll(argv[2]));
  lkv::HostTier tier;
  tier.init(0, kSlots, kFrames, kSb, 6, -1);
  Engine eng;
  std::vector<unsigned> version(kSlots, 0);  // 0 = never written / forgotten
  std::atomic<long long> mismatches{0}, checked{0};
  std::mt19937_64 rng(31);
  auto pick = [&](int n) {
    std::vector<long long> s;
    const long long base = static_cast<long long>(rng() % kSlots);
    for (int i = 0; i < n; ++i) {  // runs of neighbours with holes, like a layer's blocks
      const long long x = (base + i * (1 + static_cast<long long>(rng() % 2))) % kSlots;
      if (std::find(s.begin(), s.end(), x) == s.end()) s.push_back(x);
    }
    return s;
  };
  char* pinned = tier.pinned();
  const int steps = 6000;
  std::vector<std::vector<long long>> staged;  // staged batches not yet pinned
  for (int step = 0; step < steps; ++step) {
    if (step == steps / 3) tier.set_sticky_budget(kFrames / 3);  // resident subset, then shrunk
    if (step == 2 * steps / 3) tier.set_sticky_budget(kFrames / 12);
    const int op = static_cast<int>(rng() % 10);
    if (op < 3) {  // write (prefill pack / escalation D2H / decode append)
      auto s = pick(1 + static_cast<int>(rng() % 48));
      std::vector<long long> fr(s.size());
      tier.pin(s.data(), static_cast<long long>(s.size()), false, fr.data());
      std::vector<unsigned> ver(s.size());
      for (std::size_t i = 0; i < s.size(); ++i) ver[i] = ++version[static_cast<std::size_t>(s[i])];
      cudaEvent_t ev = stub_event_new();
      stub_event_retain(ev);
      eng.submit([=] {
        for (std::size_t i = 0; i < s.size(); ++i) {
          auto* w = reinterpret_cast<std::uint64_t*>(pinned + fr[i] * kSb);
          for (long long k = 0; k < kSb / 8; ++k) w[k] = word(s[i], ver[i], k);
        }
        stub_event_complete(ev);
        stub_event_release(ev);
      });
      tier.used(s.data(), static_cast<long long>(s.size()), ev, true);
    } else if (op < 7) {  // read (decode prefetch), staged earlier with probability 1/2
      std::vector<long long> s;
      if (!staged.empty() && rng() % 2) {
        s = staged.front();
        staged.erase(staged.begin());
      } else {
        s = pick(1 + static_cast<int>(rng() % 64));
      }
      std::vector<long long> fr(s.size());
      tier.pin(s.data(), static_cast<long long>(s.size()), true, fr.data());
      std::vector<unsigned> ver(s.size());
      for (std::size_t i = 0; i < s.size(); ++i) ver[i] = version[static_cast<std::size_t>(s[i])];
      cudaEvent_t ev = stub_event_new();
      stub_event_retain(ev);
      eng.submit([=, &mismatches, &checked] {
        for (std::size_t i = 0; i < s.size(); ++i) {
          if (ver[i] == 0) continue;  // never written: bytes undefined
          const auto* w = reinterpret_cast<const std::uint64_t*>(pinned + fr[i] * kSb);
          long long bad = 0;
          for (long long k = 0; k < kSb / 8; ++k) bad += w[k] != word(s[i], ver[i], k);
          if (bad) mismatches.fetch_add(1);
          checked.fetch_add(1);
        }
        stub_event_complete(ev);
        stub_event_release(ev);
      });
      tier.used(s.data(), static_cast<long long>(s.size()), ev, false);
    } else if (op < 9) {  // stage a batch ahead (bounded like read_ahead)
      if (staged.size() < 3) {
        auto s = pick(1 + static_cast<int>(rng() % 64));
        // a slot staged twice would pin twice: keep batches disjoint
        bool clash = false;
        for (auto& b : staged)
          for (long long x : s) clash |= std::find(b.begin(), b.end(), x) != b.end();
        if (!clash) {
          tier.stage(s.data(), static_cast<long long>(s.size()));
          staged.push_back(std::move(s));
        }
      }
    } else {  // forget (release) or unstage
      if (!staged.empty() && rng() % 2) {
        tier.unstage(staged.back().data(), static_cast<long long>(staged.back().size()));
        staged.pop_back();
      } else {
        auto s = pick(1 + static_cast<int>(rng() % 16));
        bool clash = false;  // the device never forgets a slot it has staged for the current iteration
        for (auto& b : staged)
          for (long long x : s) clash |= std::find(b.begin(), b.end(), x) != b.end();
        if (!clash) {
          tier.forget(s.data(), static_cast<long long>(s.size()));
          for (long long x : s) version[static_cast<std::size_t>(x)] = 0;
        }
      }
    }
  }
  for (auto& b : staged) tier.unstage(b.data(), static_cast<long long>(b.size()));
  // drain: every slot read back through the tier one more time
  std::vector<long long> all;
  for (long long x = 0; x < kSlots; ++x) all.push_back(x);
  for (long long x0 = 0; x0 < kSlots; x0 += 64) {
    std::vector<long long> s(all.begin() + x0, all.begin() + std::min(kSlots, x0 + 64));
    std::vector<long long> fr(s.size());
    tier.pin(s.data(), static_cast<long long>(s.size()), true, fr.data());
    for (std::size_t i = 0; i < s.size(); ++i) {
      const unsigned v = version[static_cast<std::size_t>(s[i])];
      if (!v) continue;
      const auto* w = reinterpret_cast<const std::uint64_t*>(pinned + fr[i] * kSb);
      long long bad = 0;
      for (long long k = 0; k < kSb / 8; ++k) bad += w[k] != word(s[i], v, k);
      if (bad) mismatches.fetch_add(1);
      checked.fetch_add(1);
    }
    cudaEvent_t ev = stub_event_new();
    stub_event_complete(ev);
    tier.used(s.data(), static_cast<long long>(s.size()), ev, false);
  }
  const auto st = tier.stats();
  std::printf("tier stress: %d ops, %lld frames checked, %lld mismatches; read-ins %lld, write-backs %lld, "
              "evictions %lld, staged %lld, pin waits %lld, hits %lld, resident %lld\n",
              steps, checked.load(), mismatches.load(), st.read_in_frames, st.write_back_frames, st.evictions,
              st.staged, st.pin_waits, st.hits, tier.sticky_frames());
  tier.destroy();
  return mismatches.load() == 0 && checked.load() > 0 ? 0 : 1;
}
