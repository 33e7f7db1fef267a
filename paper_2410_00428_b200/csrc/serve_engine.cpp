// Serving loop over the LayerKV data path. Event semantics
// follow the reference engine (proj/src/engine.cpp:76-453): completions of
// transfers, prefills and decode iterations, arrivals and the start tick are
// ordered by (time, kind, sequence); whenever the GPU is idle the loop admits
// (request-wise baseline, or LayerKV with the Eq. 2 SLO prefix, Eq. 5
// forecast and Half/Full escalation) and then runs one pending prefill or one
// decode iteration. The time a piece of work takes comes from the Executor:
// the modelled one below (cost model + serial PcieBus, byte-identical
// requests.csv to the reference) or the device one (serve_device.cu).
#include <algorithm>
#include <cmath>
#include <limits>
#include <queue>
#include <stdexcept>

#include "layersim/errors.hpp"
#include "layersim/prefill_span.hpp"
#include "lkv/serve.hpp"

namespace lkv {

using layersim::Direction;
using layersim::KvManager;
using layersim::OffloadMode;
using layersim::SimulationError;
using layersim::TransferJob;

// ---------------------------------------------------------------- modelled executor
ModelledExecutor::ModelledExecutor(const ServeConfig& cfg, const KvManager& kv)
    : cfg_(cfg), kv_(kv), bus_(cfg.cost.delta) {
  bus_.set_log(&log_);  // the reference keeps it under keep_transfer_log (engine.cpp:59)
}

void ModelledExecutor::count(const TransferJob& job) {
  if (job.direction == Direction::DeviceToHost) {
    ++d2h_jobs_;
    d2h_bytes_ += job.bytes;
  } else {
    ++h2d_jobs_;
    h2d_bytes_ += job.bytes;
  }
}

double ModelledExecutor::prefill(std::int64_t, std::int64_t prompt_tokens, const std::vector<int>& offloaded,
                                 double now) {
  const auto span = layersim::schedule_prefill_span(cfg_.model, cfg_.hw, cfg_.cost, bus_, offloaded, prompt_tokens,
                                                    now, cfg_.chunk_bytes, true);
  const double layer_bytes = static_cast<double>(prompt_tokens) *
                             static_cast<double>(layersim::kv_bytes_per_token_layer(cfg_.model));
  for (std::size_t i = 0; i < span.jobs.size(); ++i)
    count(TransferJob{layer_bytes, Direction::DeviceToHost, now, cfg_.chunk_bytes});
  return span.completion;
}

double ModelledExecutor::offload(const layersim::OffloadJob& job, double now) {
  const TransferJob t{job.bytes, Direction::DeviceToHost, now, cfg_.chunk_bytes};
  count(t);
  return bus_.submit_transfer(t, cfg_.hw).completion;
}

// Layer l starts when layer l-1 is done and every member's fetch of layer l
// has crossed the bus; fetches are queued in layer order at `now`
// (engine.cpp:421-449).
double ModelledExecutor::decode(const std::vector<std::int64_t>& batch, std::int64_t batch_kv_tokens, double now) {
  const int L = cfg_.model.n_layers;
  const double step = layersim::decode_step_time(cfg_.model, cfg_.hw, cfg_.cost, batch_kv_tokens);
  const double per_layer = step / L;
  const double ar = layersim::allreduce_time(cfg_.model, cfg_.hw, static_cast<std::int64_t>(batch.size()));
  std::vector<std::vector<layersim::FetchJob>> plans;
  plans.reserve(batch.size());
  for (std::int64_t id : batch) plans.push_back(kv_.plan_decode_fetch(id));
  std::vector<std::size_t> next(batch.size(), 0);
  double elapsed = 0.0;
  for (int l = 0; l < L; ++l) {
    double arrived = -1.0;
    for (std::size_t m = 0; m < plans.size(); ++m) {
      if (next[m] >= plans[m].size() || plans[m][next[m]].layer != l) continue;
      const TransferJob t{plans[m][next[m]].bytes, Direction::HostToDevice, now, cfg_.chunk_bytes};
      count(t);
      arrived = std::max(arrived, bus_.submit_transfer(t, cfg_.hw).completion);
      ++next[m];
    }
    const double begin = std::max(now + elapsed, arrived);
    elapsed = (begin - now) + per_layer;
    if (ar > 0.0) bus_.register_allreduce(now + elapsed - ar, ar, cfg_.hw);
  }
  return now + elapsed;
}

void ModelledExecutor::transfer_totals(std::int64_t* d2h_jobs, double* d2h_bytes, std::int64_t* h2d_jobs,
                                       double* h2d_bytes) const {
  *d2h_jobs = d2h_jobs_;
  *d2h_bytes = d2h_bytes_;
  *h2d_jobs = h2d_jobs_;
  *h2d_bytes = h2d_bytes_;
}

// ---------------------------------------------------------------- the loop
namespace {

enum Kind : int { kTransferDone = 0, kPrefillDone = 1, kDecodeDone = 2, kArrival = 3, kTick = 4 };

struct Ev {
  double t;
  int kind;
  std::uint64_t seq;
  std::int64_t payload;
};
struct Later {
  bool operator()(const Ev& a, const Ev& b) const {
    if (a.t != b.t) return a.t > b.t;
    if (a.kind != b.kind) return a.kind > b.kind;
    return a.seq > b.seq;
  }
};

enum class Stage { NotArrived, Waiting, Admitted, Prefilling, Decoding, Done };

struct Req {
  TraceRequest in;
  Stage stage = Stage::NotArrived;
  int retained = -1;      // x chosen at admission
  int range = -1;         // predicted output-length range
  int emitted = 0;
  double t_prefill = -1, t_first = -1, t_last = -1, t_done = -1;
};

LengthRanges ranges_for(const Trace& t, double accuracy) {
  std::vector<int> out;
  out.reserve(t.requests.size());
  for (const TraceRequest& r : t.requests) out.push_back(r.output_tokens);
  return LengthRanges::deciles(std::move(out), accuracy);
}

}  // namespace

struct ServeEngine::Impl {
  ServeConfig cfg;
  KvManager& kv;
  Executor* exec = nullptr;
  LengthRanges ranges;
  std::vector<Req> reqs;
  std::priority_queue<Ev, std::vector<Ev>, Later> events;
  std::uint64_t seq = 0;
  std::vector<std::int64_t> waiting;   // arrived, not admitted (FCFS); front = index `waiting_head`
  std::size_t waiting_head = 0;
  std::vector<std::int64_t> to_prefill;  // admitted, awaiting the GPU (FCFS)
  std::size_t prefill_head = 0;
  std::vector<std::int64_t> decoding;  // by first token
  std::vector<std::int64_t> live;      // admitted and unfinished (any order)
  std::vector<std::int64_t> in_batch;
  bool busy = false;
  std::int64_t escalations = 0;
  std::vector<DecisionRecord> decisions;  // LayerKV admission rounds (decision_log.csv)
  std::int64_t threshold = 0;
  int done = 0;

  Impl(ServeConfig c, const Trace& trace, KvManager& k)
      : cfg(std::move(c)), kv(k), ranges(ranges_for(trace, cfg.predictor_accuracy)) {}

  void push(double t, int kind, std::int64_t payload) { events.push({t, kind, seq++, payload}); }
  std::size_t n_waiting() const { return waiting.size() - waiting_head; }
  std::int64_t waiting_at(std::size_t k) const { return waiting[waiting_head + k]; }
  Req& R(std::int64_t i) { return reqs[static_cast<std::size_t>(i)]; }
  int L() const { return cfg.model.n_layers; }
  int tpb() const { return kv.tokens_per_block(); }
  std::int64_t rows_for(std::int64_t tokens) const { return (tokens + tpb() - 1) / tpb() + 1; }

  // ---- events
  void arrive(std::int64_t i) {
    Req& r = R(i);
    r.stage = Stage::Waiting;
    Splitmix draws = Splitmix::keyed(cfg.seed, "predictor", static_cast<std::uint64_t>(i));
    r.range = ranges.predict(r.in.output_tokens, draws);
    waiting.push_back(i);
  }

  void finish(std::int64_t i, double now) {
    Req& r = R(i);
    r.stage = Stage::Done;
    r.t_done = now;
    exec->before_release(i);
    kv.release(i);
    decoding.erase(std::remove(decoding.begin(), decoding.end(), i), decoding.end());
    live.erase(std::remove(live.begin(), live.end(), i), live.end());
    ++done;
  }

  void prefill_done(std::int64_t i, double now) {
    Req& r = R(i);
    r.t_first = r.t_last = now;
    r.emitted = 1;
    busy = false;
    if (r.in.output_tokens == 1) {
      finish(i, now);
    } else {
      r.stage = Stage::Decoding;
      decoding.push_back(i);
    }
  }

  void decode_done(double now) {
    busy = false;
    std::vector<std::int64_t> finished;
    for (std::int64_t i : in_batch) {
      Req& r = R(i);
      kv.note_token(i);
      ++r.emitted;
      r.t_last = now;
      if (r.emitted >= r.in.output_tokens) finished.push_back(i);
    }
    in_batch.clear();
    for (std::int64_t i : finished) finish(i, now);
  }

  // ---- admission helpers
  void reserve_rows(std::int64_t* gpu, std::int64_t* cpu) const {
    std::int64_t g = 0, c = 0;
    for (std::int64_t i : live) {
      const Req& r = reqs[static_cast<std::size_t>(i)];
      const std::int64_t rows = rows_for(std::max(0, r.in.output_tokens - r.emitted));
      g += rows * kv.gpu_row_cost(i);
      c += rows * kv.cpu_row_cost(i);
    }
    *gpu = g;
    *cpu = c;
  }

  // A head that cannot fit even into empty, idle pools can never run
  // (engine.cpp:188-210).
  void never_fits_check(std::int64_t i) const {
    if (!decoding.empty() || prefill_head < to_prefill.size() || busy) return;
    if (kv.gpu_blocks_free() != kv.gpu_blocks_total() || kv.cpu_blocks_free() != kv.cpu_blocks_total()) return;
    const Req& r = reqs[static_cast<std::size_t>(i)];
    const std::int64_t all = kv.blocks_per_layer(r.in.prompt_tokens) * L();
    const bool too_big = cfg.layerkv ? all > kv.cpu_blocks_total() : all > kv.gpu_blocks_total();
    if (too_big)
      throw SimulationError("engine: request " + std::to_string(i) + " can never be admitted (prompt " +
                            std::to_string(r.in.prompt_tokens) + " tokens exceeds pool capacity)");
  }

  void admit(std::int64_t i, int x) {
    ++waiting_head;
    Req& r = R(i);
    r.stage = Stage::Admitted;
    r.retained = x;
    to_prefill.push_back(i);
    live.push_back(i);
  }

  void admit_request_wise() {
    while (n_waiting() > 0) {
      const std::int64_t i = waiting_at(0);
      const Req& r = R(i);
      std::int64_t res_gpu = 0, res_cpu = 0;
      reserve_rows(&res_gpu, &res_cpu);
      res_gpu += rows_for(r.in.output_tokens) * L();
      if (kv.gpu_blocks_free() < kv.request_wise_gpu_blocks(r.in.prompt_tokens) + res_gpu) {
        never_fits_check(i);
        return;
      }
      if (!kv.allocate_prefill(i, r.in.prompt_tokens, L())) return;
      admit(i, L());
    }
  }

  int layers_to_retain(std::int64_t prompt, bool pressured) const {
    if (cfg.force_retained_layers >= 0) return std::min(cfg.force_retained_layers, L());
    if (!pressured) return L();
    return layersim::min_retained_layers(cfg.model, cfg.hw, cfg.cost, prompt);
  }

  void admit_layerwise(double now) {
    // Eq. 2 slack of every request past its first decode token.
    std::vector<double> slack;
    for (std::int64_t i : decoding) {
      const Req& r = R(i);
      const std::int64_t n_past = r.emitted - 1;
      if (n_past >= 1) slack.push_back(prefill_slack(now - r.t_first, n_past, ranges.lo(r.range), cfg.slo));
    }
    double min_budget = std::numeric_limits<double>::infinity();
    for (double b : slack) min_budget = std::min(min_budget, b);
    int n;
    if (cfg.slo_scheduler) {
      std::vector<double> cost;
      cost.reserve(n_waiting());
      for (std::size_t k = 0; k < n_waiting(); ++k)
        cost.push_back(layersim::prefill_time(cfg.model, cfg.hw, cfg.cost, R(waiting_at(k)).in.prompt_tokens));
      double committed = 0.0;
      for (std::size_t k = prefill_head; k < to_prefill.size(); ++k)
        committed += layersim::prefill_time(cfg.model, cfg.hw, cfg.cost, R(to_prefill[k]).in.prompt_tokens);
      n = admissible_prefix(cost, slack, committed);
    } else {
      n = static_cast<int>(n_waiting());
    }

    // Eq. 5 forecast with the planned admissions' request-wise demand.
    std::int64_t planned = 0;
    for (int k = 0; k < n; ++k) planned += kv.request_wise_gpu_blocks(R(waiting_at(static_cast<std::size_t>(k))).in.prompt_tokens);
    std::vector<HeldForecast> held;
    held.reserve(decoding.size());
    std::int64_t reclaim_half = 0, reclaim_full = 0;
    for (std::int64_t i : decoding) {
      const Req& r = R(i);
      const std::int64_t median = (static_cast<std::int64_t>(ranges.lo(r.range)) + ranges.hi(r.range)) / 2;
      held.push_back({kv.gpu_blocks_held(i), std::max<std::int64_t>(0, median - r.emitted)});
      reclaim_half += kv.offload_reclaim(i, OffloadMode::Half);
      reclaim_full += kv.offload_reclaim(i, OffloadMode::Full);
    }
    const std::vector<double> fc =
        availability_forecast(static_cast<double>(kv.gpu_blocks_free()), cfg.horizon, held, planned, n);
    const Escalation esc = escalation_for(fc, static_cast<double>(threshold), reclaim_half);

    if (esc != Escalation::None) {
      const double low = *std::min_element(fc.begin(), fc.end());
      const std::int64_t needed = threshold - static_cast<std::int64_t>(low);
      // Most recent first token first; ties by larger index.
      std::vector<std::int64_t> victims(decoding);
      std::sort(victims.begin(), victims.end(), [this](std::int64_t a, std::int64_t b) {
        const double fa = R(a).t_first, fb = R(b).t_first;
        return fa != fb ? fa > fb : a > b;
      });
      const OffloadMode mode = esc == Escalation::Half ? OffloadMode::Half : OffloadMode::Full;
      std::int64_t credited = 0;
      for (std::int64_t i : victims) {
        if (credited >= needed) break;
        const auto job = kv.plan_offload(i, mode);
        if (!job) break;            // CPU pool exhausted
        if (job->job_id < 0) continue;  // nothing retained
        ++escalations;
        const double t = exec->offload(*job, now);
        if (!std::isnan(t)) push(t, kTransferDone, job->job_id);  // NaN: measured, reported by poll_offloads
        credited += job->gpu_blocks;
      }
    }

    int admitted = 0;
    // logged like engine.cpp:388-390, also when an admission stops the round
    const auto log_decision = [&] {
      if (admitted > 0 || esc != Escalation::None) decisions.push_back({now, min_budget, admitted, esc});
    };
    for (int k = 0; k < n && n_waiting() > 0; ++k) {
      const std::int64_t i = waiting_at(0);
      const Req& r = R(i);
      std::int64_t res_gpu = 0, res_cpu = 0;
      reserve_rows(&res_gpu, &res_cpu);
      const std::int64_t per_layer = kv.blocks_per_layer(r.in.prompt_tokens);
      const std::int64_t own = rows_for(r.in.output_tokens);
      const auto fits = [&](int x) {
        const std::int64_t off = L() - x;
        return kv.gpu_blocks_free() >= per_layer * x + own * x + res_gpu &&
               kv.cpu_blocks_free() >= per_layer * off + own * off + res_cpu;
      };
      int x = layers_to_retain(r.in.prompt_tokens, esc != Escalation::None);
      bool ok = fits(x) && kv.allocate_prefill(i, r.in.prompt_tokens, x);
      if (!ok && x == L() && cfg.force_retained_layers < 0) {  // forecast missed: overlap-safe minimum
        x = layersim::min_retained_layers(cfg.model, cfg.hw, cfg.cost, r.in.prompt_tokens);
        ok = fits(x) && kv.allocate_prefill(i, r.in.prompt_tokens, x);
      }
      if (!ok) {
        never_fits_check(i);
        log_decision();
        return;
      }
      admit(i, x);
      ++admitted;
    }
    log_decision();
  }

  // ---- GPU work
  void run_prefill(std::int64_t i, double now) {
    Req& r = R(i);
    r.stage = Stage::Prefilling;
    r.t_prefill = now;
    busy = true;
    const layersim::PlacementPlan plan = layersim::layer_placement(L(), r.retained);
    push(exec->prefill(i, r.in.prompt_tokens, plan.offloaded, now), kPrefillDone, i);
  }

  void run_decode(double now) {
    in_batch.clear();
    std::int64_t kv_tokens = 0;
    for (std::int64_t i : decoding) {
      if (kv.needs_append(i) && !kv.append_decode_block(i)) continue;  // sits this iteration out
      const std::int64_t t = kv.request(i).cached_tokens;
      if (!in_batch.empty() && kv_tokens + t > cfg.max_batch_tokens) break;  // FCFS cap
      in_batch.push_back(i);
      kv_tokens += t;
    }
    if (in_batch.empty()) return;
    busy = true;
    push(exec->decode(in_batch, kv_tokens, now), kDecodeDone, -1);
  }

  void schedule(double now) {
    if (busy) return;
    if (cfg.layerkv)
      admit_layerwise(now);
    else
      admit_request_wise();
    if (prefill_head < to_prefill.size()) {
      run_prefill(to_prefill[prefill_head++], now);
      return;
    }
    if (!decoding.empty()) run_decode(now);
  }

  ServeReport loop() {
    double now = 0.0;
    bool completed = true;
    const bool measured = exec->measured();
    std::vector<std::pair<double, std::int64_t>> landed;
    for (;;) {
      if (measured) {
        // Every offload that completes before the next event must be in the
        // queue first: poll, and block on the oldest while the next event
        // lies beyond the hardware's present.
        exec->poll_offloads(false, &landed);
        while (exec->offloads_pending() && (events.empty() || events.top().t > exec->clock()))
          exec->poll_offloads(true, &landed);
        for (const auto& [t, job] : landed) push(t, kTransferDone, job);
        landed.clear();
      }
      if (events.empty()) break;
      const Ev e = events.top();
      events.pop();
      if (e.t > cfg.max_time) {
        completed = false;
        now = cfg.max_time;
        break;
      }
      if (measured && e.t > exec->clock()) exec->skip_to(e.t);  // idle until the next arrival
      now = e.t;
      switch (e.kind) {
        case kArrival: arrive(e.payload); break;
        case kPrefillDone: prefill_done(e.payload, now); break;
        case kDecodeDone: decode_done(now); break;
        case kTransferDone: kv.complete_offload(e.payload); break;
        default: break;
      }
      if (cfg.invariant_checks) kv.check_conservation();
      if (!busy) schedule(now);
    }
    if (completed && done != static_cast<int>(reqs.size()))
      throw SimulationError("engine: no runnable work left with " + std::to_string(reqs.size() - done) +
                            " unfinished requests (block starvation); queued=" + std::to_string(n_waiting()) +
                            " pending_prefill=" + std::to_string(to_prefill.size() - prefill_head) +
                            " decoding=" + std::to_string(decoding.size()) + " gpu_free=" +
                            std::to_string(kv.gpu_blocks_free()) + "/" + std::to_string(kv.gpu_blocks_total()) +
                            " cpu_free=" + std::to_string(kv.cpu_blocks_free()) + "/" +
                            std::to_string(kv.cpu_blocks_total()) + " t=" + std::to_string(now));
    std::vector<RequestRecord> rows;
    double makespan = 0.0;
    for (const Req& r : reqs) {
      if (r.stage != Stage::Done) continue;
      RequestRecord m;
      m.id = r.in.id;
      m.arrival = r.in.arrival;
      m.queuing = r.t_prefill - r.in.arrival;
      m.prefill = r.t_first - r.t_prefill;
      m.ttft = m.queuing + m.prefill;
      m.output_tokens = r.in.output_tokens;
      m.mean_tpot = r.in.output_tokens > 1 ? (r.t_last - r.t_first) / (r.in.output_tokens - 1) : 0.0;
      rows.push_back(m);
      makespan = std::max(makespan, r.t_done);
    }
    if (!completed) makespan = now;
    ServeReport rep = ServeReport::summarize(std::move(rows), makespan, completed, cfg.slo);
    exec->transfer_totals(&rep.d2h_jobs, &rep.d2h_bytes, &rep.h2d_jobs, &rep.h2d_bytes);
    if (const auto* log = exec->transfer_log()) rep.transfer_log = *log;
    rep.escalations = escalations;
    rep.decision_log = decisions;
    return rep;
  }
};

ServeEngine::ServeEngine(ServeConfig cfg, Trace trace, ExecutorFactory make_executor) {
  cfg.model.validate();
  cfg.hw.validate();
  cfg.cost.validate();
  if (cfg.slo.ttft <= 0.0 || cfg.slo.tpot <= 0.0) throw std::invalid_argument("SLOSpec: thresholds must be positive");
  trace.validate();
  kv_ = std::make_unique<KvManager>(cfg.pools, cfg.model);
  impl_ = std::make_unique<Impl>(cfg, trace, *kv_);
  exec_ = make_executor ? make_executor(impl_->cfg, *kv_) : std::make_unique<ModelledExecutor>(impl_->cfg, *kv_);
  impl_->exec = exec_.get();
  impl_->threshold =
      static_cast<std::int64_t>(impl_->cfg.threshold_fraction * static_cast<double>(impl_->cfg.pools.gpu_blocks_total));
  impl_->reqs.reserve(trace.requests.size());
  for (const TraceRequest& t : trace.requests) {
    Req r;
    r.in = t;
    impl_->reqs.push_back(r);
    impl_->push(t.arrival, kArrival, static_cast<std::int64_t>(impl_->reqs.size()) - 1);
  }
  impl_->push(0.0, kTick, -1);
}

ServeEngine::~ServeEngine() {
  impl_.reset();
  exec_.reset();  // the executor (device observer) goes before the manager
  kv_.reset();
}

ServeReport ServeEngine::run() { return impl_->loop(); }

}  // namespace lkv
