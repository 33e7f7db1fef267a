// Serving layer around the LayerKV data path.
//
// The reference's caller of the hot path is a discrete-event engine
// (proj/src/engine.cpp) with an SLO-aware admission scheduler
// (proj/src/scheduler.cpp), synthetic/JSONL traces (proj/src/workload.cpp)
// and per-request metrics (proj/src/metrics.cpp). This header restates those
// as one B200-side serving loop whose time source is pluggable:
//
//   * Clock "virtual"  — durations from the reference cost model and the
//     serial PcieBus (cost_model.cpp, interconnect.cpp). With the same trace
//     and config it reproduces the reference's requests.csv byte for byte
//     (tests/test_serve_engine.py against tests/golden/engine.json). The
//     device may execute the same jobs underneath without touching the clock.
//   * Clock "measured" — every prefill, decode iteration and escalation D2H
//     runs on the GPU (liblkv device path + cuBLAS dense GEMMs) and its
//     CUDA-event duration advances the clock; idle gaps jump to the next
//     arrival. TTFT/TPOT are then measured, not modelled.
//
// Only the loop, the scheduler math and the formats live here; KV state is
// the drop-in layersim::KvManager and the data path is lkv_device.
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <string_view>
#include <vector>

#include "layersim/cost_model.hpp"
#include "layersim/interconnect.hpp"
#include "layersim/kv_manager.hpp"

namespace lkv {

// ---------------------------------------------------------------- draws
// splitmix64 stream with hand-rolled distributions, identical draws to the
// reference Rng (rng.hpp:12-69) so traces and predictor outcomes agree bit
// for bit (the reference chose it to be platform-stable).
class Splitmix {
 public:
  explicit Splitmix(std::uint64_t seed) : s_(seed) {}
  // Stream keyed by (seed, label, index): FNV-1a of the label mixed into the
  // seed, offset by the golden-ratio step per index, two draws discarded.
  static Splitmix keyed(std::uint64_t seed, std::string_view label, std::uint64_t index = 0);
  std::uint64_t next();
  double unit();                      // [0, 1), 53 bits
  double exponential(double mean);    // -mean * log1p(-u)
  double lognormal(double mu, double sigma);  // exp of Box-Muller (two uniforms, no spare)

 private:
  std::uint64_t s_;
};

// ---------------------------------------------------------------- traces (f4)
struct TraceRequest {
  std::int64_t id = 0;
  double arrival = 0.0;    // seconds from start
  int prompt_tokens = 0;
  int output_tokens = 0;   // true length; the scheduler sees it only through the predictor
};

struct Trace {
  std::vector<TraceRequest> requests;  // ascending arrival
  std::uint64_t seed = 0;
  void validate() const;               // std::invalid_argument, as workload.cpp:15-33
};

// Poisson arrivals at `rate`, fixed lengths (workload.cpp:35-52).
Trace trace_fixed(int n, int prompt_tokens, int output_tokens, double rate, std::uint64_t seed);
// Poisson arrivals, log-normal(mu, sigma) lengths rounded and clamped to
// [min_len, max_len] for prompt then output (workload.cpp:54-82).
Trace trace_sharegpt_like(int n, double rate, std::uint64_t seed, double mu = 5.0, double sigma = 1.0,
                          int min_len = 4, int max_len = 2300);
// JSONL: one object per line with arrival_s, prompt_tokens, output_tokens
// (optional id), '#' comments; unsorted input is stable-sorted and flagged;
// malformed lines raise std::runtime_error naming path:line
// (workload.cpp:84-136). Writer emits {"id","arrival_s","prompt_tokens",
// "output_tokens"} per line with shortest round-trip doubles.
Trace read_trace_jsonl(const std::string& path, bool* was_unsorted = nullptr);
std::string trace_to_jsonl(const Trace& trace);
void write_trace_jsonl(const Trace& trace, const std::string& path);

// ---------------------------------------------------------------- SLO scheduler
struct Slo {
  double ttft = 3.0;  // s
  double tpot = 0.2;  // s per token
};

// Output-length ranges [edge_i, edge_{i+1}); edges start at 1 and end at
// max_len + 1 (scheduler.hpp:22-44).
class LengthRanges {
 public:
  LengthRanges(std::vector<int> interior, int max_len, double accuracy);
  static LengthRanges deciles(std::vector<int> lengths, double accuracy);
  int count() const { return static_cast<int>(edges_.size()) - 1; }
  int lo(int i) const { return edges_[static_cast<std::size_t>(i)]; }
  int hi(int i) const { return edges_[static_cast<std::size_t>(i) + 1]; }
  int index_of(int length) const;
  double accuracy() const { return accuracy_; }
  // Predictor stand-in: the true range with probability `accuracy`, else a
  // neighbour (clamped at the ends) — scheduler.cpp:68-79.
  int predict(int true_len, Splitmix& draws) const;

 private:
  std::vector<int> edges_;
  double accuracy_;
};

// Eq. 2 slack of one decoding request (scheduler.cpp:81-96).
double prefill_slack(double t_past, std::int64_t n_past, int predicted_lo, const Slo& slo);
// Largest queue prefix whose cumulative prefill time (after `committed`)
// stays strictly below every slack (scheduler.cpp:98-111).
int admissible_prefix(const std::vector<double>& prefill_times, const std::vector<double>& slacks,
                      double committed);
struct HeldForecast {
  std::int64_t gpu_blocks = 0;
  std::int64_t stages_left = 0;
};
// Eq. 5 availability series Avail(0..horizon) (scheduler.cpp:113-138).
std::vector<double> availability_forecast(double avail0, int horizon, const std::vector<HeldForecast>& decoding,
                                          std::int64_t planned_blocks, int planned_count);
enum class Escalation { None, Half, Full };
Escalation escalation_for(const std::vector<double>& forecast, double threshold, std::int64_t reclaim_half);

// ---------------------------------------------------------------- metrics (f4)
struct RequestRecord {
  std::int64_t id = 0;
  double arrival = 0.0, queuing = 0.0, prefill = 0.0, ttft = 0.0, mean_tpot = 0.0;
  int output_tokens = 0;
  bool violated = false, violated_ttft = false, violated_tpot = false;
};

// One LayerKV admission round that admitted or escalated (the reference's
// DecisionLogRow, engine.hpp:52-57, recorded at engine.cpp:388-390).
struct DecisionRecord {
  double time = 0.0;
  double min_budget = 0.0;  // smallest Eq. 2 slack; +inf when no decoding request constrains it
  int admitted = 0;
  Escalation plan = Escalation::None;
};

struct ServeReport {
  std::vector<RequestRecord> requests;  // ascending id
  double mean_ttft = 0, p50_ttft = 0, p99_ttft = 0, mean_tpot = 0, mean_queuing = 0, mean_prefill = 0;
  double queuing_fraction = 0, throughput_tokens_per_s = 0, violation_rate = 0, makespan = 0;
  int violations = 0, violations_ttft = 0, violations_tpot = 0;
  std::int64_t total_output_tokens = 0;
  bool completed = true;
  // transfer totals (jobs / bytes per direction) over the run
  std::int64_t d2h_jobs = 0, h2d_jobs = 0;
  double d2h_bytes = 0, h2d_bytes = 0;
  std::int64_t escalations = 0;  // plan_offload jobs submitted (engine.cpp:343-352)
  // every bus transfer of the virtual clock in submission order (the
  // reference's Engine::transfer_log, interconnect.hpp:26-33); empty under the
  // measured clock
  std::vector<layersim::TransferLogRow> transfer_log;
  std::vector<DecisionRecord> decision_log;  // LayerKV policy only

  static ServeReport summarize(std::vector<RequestRecord> rows, double makespan, bool completed, const Slo& slo);
  std::string requests_csv() const;  // metrics.cpp:91-101 format, "%.9g"
  std::string summary_json() const;  // metrics.cpp:69-88 keys
  // transfer_log.csv of the reference CLI (tools/layersim_main.cpp:96-105)
  std::string transfer_log_csv() const;
  // decision_log.csv of the reference CLI (tools/layersim_main.cpp:107-117)
  std::string decision_log_csv() const;
};
std::string fmt9(double v);                         // "%.9g"
double nearest_rank(std::vector<double> v, double q);  // metrics.cpp:22-29

// ---------------------------------------------------------------- executor
// What the loop asks the hardware (or the model of it) to do. Each call
// returns the completion time on the engine's clock.
class Executor {
 public:
  virtual ~Executor() = default;
  // Prefill of `id`: layer l's K/V are produced and scattered (retained) or
  // packed + D2H'd (offloaded, ascending `offloaded`).
  virtual double prefill(std::int64_t id, std::int64_t prompt_tokens, const std::vector<int>& offloaded,
                         double now) = 0;
  // Escalation D2H of a planned offload job (engine.cpp:343-352).
  virtual double offload(const layersim::OffloadJob& job, double now) = 0;
  // One decode iteration over `batch` (every member already appended its
  // block if needed); fetches per member are plan_decode_fetch's.
  virtual double decode(const std::vector<std::int64_t>& batch, std::int64_t batch_kv_tokens, double now) = 0;
  // Transfer totals so far.
  virtual void transfer_totals(std::int64_t* d2h_jobs, double* d2h_bytes, std::int64_t* h2d_jobs,
                               double* h2d_bytes) const = 0;
  // The virtual clock's bus transfers so far (nullptr: none kept).
  virtual const std::vector<layersim::TransferLogRow>* transfer_log() const { return nullptr; }
  // The request's KV is about to be released (its slots return to the pools).
  virtual void before_release(std::int64_t /*id*/) {}

  // ---- measured clocks only. offload() may then return NaN: the job's
  // completion is learned from the hardware and reported by poll_offloads.
  virtual bool measured() const { return false; }
  virtual double clock() { return 0.0; }          // engine time now
  virtual void skip_to(double /*t*/) {}           // idle: jump the clock to t
  virtual bool offloads_pending() const { return false; }
  // Completed jobs as (time, job id), oldest first; `wait` blocks for the
  // oldest pending job.
  virtual void poll_offloads(bool /*wait*/, std::vector<std::pair<double, std::int64_t>>* /*done*/) {}
};

struct ServeConfig {
  layersim::ModelSpec model;
  layersim::HardwareSpec hw;
  layersim::CostParams cost;
  Slo slo;
  bool layerkv = true;                 // false: request-wise baseline
  bool slo_scheduler = true;           // layerkv only
  layersim::BlockPools pools;
  double threshold_fraction = 0.05;
  int horizon = 8;
  double predictor_accuracy = 0.8;
  std::int64_t max_batch_tokens = 131072;
  double max_time = 86400.0;
  double chunk_bytes = 16.0 * 1024 * 1024;
  std::uint64_t seed = 0;
  int force_retained_layers = -1;
  bool invariant_checks = false;
};

// Virtual clock: reference cost model + serial PcieBus.
class ModelledExecutor final : public Executor {
 public:
  ModelledExecutor(const ServeConfig& cfg, const layersim::KvManager& kv);
  double prefill(std::int64_t id, std::int64_t prompt_tokens, const std::vector<int>& offloaded,
                 double now) override;
  double offload(const layersim::OffloadJob& job, double now) override;
  double decode(const std::vector<std::int64_t>& batch, std::int64_t batch_kv_tokens, double now) override;
  void transfer_totals(std::int64_t* d2h_jobs, double* d2h_bytes, std::int64_t* h2d_jobs,
                       double* h2d_bytes) const override;
  const std::vector<layersim::TransferLogRow>* transfer_log() const override { return &log_; }
  layersim::PcieBus& bus() { return bus_; }

 private:
  void count(const layersim::TransferJob& job);
  const ServeConfig& cfg_;
  const layersim::KvManager& kv_;
  layersim::PcieBus bus_;
  std::vector<layersim::TransferLogRow> log_;  // bus_ appends every transfer
  std::int64_t d2h_jobs_ = 0, h2d_jobs_ = 0;
  double d2h_bytes_ = 0, h2d_bytes_ = 0;
};

class ServeEngine {
 public:
  // `make_executor` receives the engine's KvManager (so a device executor can
  // bind to it). nullptr → ModelledExecutor.
  using ExecutorFactory = std::function<std::unique_ptr<Executor>(const ServeConfig&, layersim::KvManager&)>;
  ServeEngine(ServeConfig cfg, Trace trace, ExecutorFactory make_executor = nullptr);
  ~ServeEngine();
  ServeReport run();
  const layersim::KvManager& kv() const { return *kv_; }
  Executor& executor() { return *exec_; }

 private:
  struct Impl;
  std::unique_ptr<layersim::KvManager> kv_;
  std::unique_ptr<Executor> exec_;
  std::unique_ptr<Impl> impl_;
};

}  // namespace lkv
