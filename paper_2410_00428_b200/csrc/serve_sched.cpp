// SLO-aware admission math and per-request metrics of the serving loop.
// Host logic only (north star: "the SLO-aware scheduler remains host logic
// and only drives the device path"). Restates proj/src/scheduler.cpp and
// proj/src/metrics.cpp with the same arithmetic order, so the virtual clock
// reproduces the reference's requests.csv byte for byte.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <sstream>
#include <stdexcept>

#include "lkv/serve.hpp"

namespace lkv {

// ---------------------------------------------------------------- length ranges
LengthRanges::LengthRanges(std::vector<int> interior, int max_len, double accuracy) : accuracy_(accuracy) {
  if (!(accuracy >= 0.0 && accuracy <= 1.0)) throw std::invalid_argument("LengthBuckets: accuracy must be in [0, 1]");
  edges_.reserve(interior.size() + 2);
  edges_.push_back(1);
  for (int b : interior) {
    if (b <= edges_.back()) throw std::invalid_argument("LengthBuckets: boundaries must be strictly increasing");
    edges_.push_back(b);
  }
  if (max_len + 1 <= edges_.back()) throw std::invalid_argument("LengthBuckets: max_len below last boundary");
  edges_.push_back(max_len + 1);
}

// Deciles k/10 of the sorted sample; a boundary must exceed 1, the sample
// minimum and the previous boundary, and not exceed the maximum
// (scheduler.cpp:33-52).
LengthRanges LengthRanges::deciles(std::vector<int> lengths, double accuracy) {
  if (lengths.empty()) throw std::invalid_argument("LengthBuckets: empty length sample");
  std::sort(lengths.begin(), lengths.end());
  const std::size_t n = lengths.size();
  const int smallest = lengths.front(), largest = lengths.back();
  std::vector<int> cuts;
  for (std::size_t k = 1; k < 10; ++k) {
    const int b = lengths[std::min(k * n / 10, n - 1)];
    const bool fresh = cuts.empty() || b > cuts.back();
    if (b > 1 && b > smallest && b <= largest && fresh) cuts.push_back(b);
  }
  return LengthRanges(std::move(cuts), largest, accuracy);
}

int LengthRanges::index_of(int length) const {
  const int k = count();
  for (int i = 0; i < k; ++i)
    if (length < hi(i)) return i;
  return k - 1;
}

int LengthRanges::predict(int true_len, Splitmix& draws) const {
  if (true_len < 1) throw std::invalid_argument("predict_bucket: length must be >= 1");
  const int truth = index_of(true_len);
  const int k = count();
  if (k == 1 || draws.unit() < accuracy_) return truth;
  if (truth == 0) return 1;
  if (truth == k - 1) return truth - 1;
  return draws.unit() < 0.5 ? truth - 1 : truth + 1;
}

// ---------------------------------------------------------------- Eq. 2 / Eq. 5
double prefill_slack(double t_past, std::int64_t n_past, int predicted_lo, const Slo& slo) {
  if (n_past < 1) throw std::invalid_argument("allow_prefill_budget: n_past must be >= 1");
  const double future = static_cast<double>(std::max<std::int64_t>(1, predicted_lo - n_past));
  const double per_token = t_past / static_cast<double>(n_past);
  const double t_future = per_token * future;
  return slo.tpot * (static_cast<double>(n_past) + future) - (t_past + t_future);
}

int admissible_prefix(const std::vector<double>& prefill_times, const std::vector<double>& slacks, double committed) {
  double tightest = std::numeric_limits<double>::infinity();
  for (double s : slacks) tightest = std::min(tightest, s);
  double total = committed;
  int n = 0;
  for (double t : prefill_times) {
    total += t;
    if (!(total < tightest)) break;
    ++n;
  }
  return n;
}

std::vector<double> availability_forecast(double avail0, int horizon, const std::vector<HeldForecast>& decoding,
                                          std::int64_t planned_blocks, int planned_count) {
  if (horizon < 1) throw std::invalid_argument("forecast_availability: horizon must be >= 1");
  std::vector<double> a(static_cast<std::size_t>(horizon) + 1);
  a[0] = avail0;
  for (int t = 0; t < horizon; ++t) {
    double freed = 0.0, growing = 0.0;
    for (const HeldForecast& s : decoding) {
      if (s.stages_left == t) freed += static_cast<double>(s.gpu_blocks);
      if (s.stages_left > t) growing += 1.0;
    }
    const double taken = growing + (t == 0 ? static_cast<double>(planned_blocks) : static_cast<double>(planned_count));
    a[static_cast<std::size_t>(t) + 1] = a[static_cast<std::size_t>(t)] + freed - taken;
  }
  return a;
}

Escalation escalation_for(const std::vector<double>& forecast, double threshold, std::int64_t reclaim_half) {
  double low = std::numeric_limits<double>::infinity();
  for (double v : forecast) low = std::min(low, v);
  if (low >= threshold) return Escalation::None;
  return low + static_cast<double>(reclaim_half) >= threshold ? Escalation::Half : Escalation::Full;
}

// ---------------------------------------------------------------- metrics
std::string fmt9(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.9g", v);
  return buf;
}

double nearest_rank(std::vector<double> v, double q) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  auto r = static_cast<std::size_t>(std::ceil(q * static_cast<double>(v.size())));
  r = std::clamp<std::size_t>(r, 1, v.size());
  return v[r - 1];
}

ServeReport ServeReport::summarize(std::vector<RequestRecord> rows, double makespan, bool completed, const Slo& slo) {
  ServeReport rep;
  rep.makespan = makespan;
  rep.completed = completed;
  std::sort(rows.begin(), rows.end(), [](const RequestRecord& a, const RequestRecord& b) { return a.id < b.id; });
  rep.requests = std::move(rows);
  if (rep.requests.empty()) return rep;
  std::vector<double> ttft;
  ttft.reserve(rep.requests.size());
  double s_ttft = 0.0, s_tpot = 0.0, s_q = 0.0, s_p = 0.0;
  for (RequestRecord& r : rep.requests) {
    r.violated_ttft = r.ttft > slo.ttft;
    r.violated_tpot = r.output_tokens > 1 && r.mean_tpot > slo.tpot;
    r.violated = r.violated_ttft || r.violated_tpot;
    ttft.push_back(r.ttft);
    s_ttft += r.ttft;
    s_tpot += r.mean_tpot;
    s_q += r.queuing;
    s_p += r.prefill;
    rep.total_output_tokens += r.output_tokens;
    rep.violations += r.violated;
    rep.violations_ttft += r.violated_ttft;
    rep.violations_tpot += r.violated_tpot;
  }
  const double n = static_cast<double>(rep.requests.size());
  rep.mean_ttft = s_ttft / n;
  rep.mean_tpot = s_tpot / n;
  rep.mean_queuing = s_q / n;
  rep.mean_prefill = s_p / n;
  rep.queuing_fraction = rep.mean_ttft > 0.0 ? rep.mean_queuing / rep.mean_ttft : 0.0;
  rep.p50_ttft = nearest_rank(ttft, 0.50);
  rep.p99_ttft = nearest_rank(ttft, 0.99);
  rep.violation_rate = rep.violations / n;
  rep.throughput_tokens_per_s = makespan > 0.0 ? static_cast<double>(rep.total_output_tokens) / makespan : 0.0;
  return rep;
}

std::string ServeReport::requests_csv() const {
  std::ostringstream os;
  os << "id,arrival,queuing_s,prefill_s,ttft_s,mean_tpot_s,output_tokens,violated\n";
  for (const RequestRecord& r : requests)
    os << r.id << ',' << fmt9(r.arrival) << ',' << fmt9(r.queuing) << ',' << fmt9(r.prefill) << ',' << fmt9(r.ttft)
       << ',' << fmt9(r.mean_tpot) << ',' << r.output_tokens << ',' << (r.violated ? 1 : 0) << '\n';
  return os.str();
}

std::string ServeReport::transfer_log_csv() const {
  std::ostringstream os;
  os << "submit_s,start_s,end_s,bytes,direction,deferrals\n";
  for (const layersim::TransferLogRow& t : transfer_log)
    os << fmt9(t.submit) << ',' << fmt9(t.start) << ',' << fmt9(t.end) << ',' << fmt9(t.bytes) << ','
       << (t.direction == layersim::Direction::DeviceToHost ? "d2h" : "h2d") << ',' << t.deferrals << '\n';
  return os.str();
}

std::string ServeReport::decision_log_csv() const {
  std::ostringstream os;
  os << "time_s,min_budget_s,admitted,offload_plan\n";
  for (const DecisionRecord& d : decision_log)
    os << fmt9(d.time) << ',' << fmt9(d.min_budget) << ',' << d.admitted << ','
       << (d.plan == Escalation::None ? "none" : d.plan == Escalation::Half ? "half" : "full") << '\n';
  return os.str();
}

std::string ServeReport::summary_json() const {
  std::ostringstream os;
  os << "{\n  \"requests\": " << requests.size() << ",\n  \"completed\": " << (completed ? "true" : "false")
     << ",\n  \"mean_ttft_s\": " << fmt9(mean_ttft) << ",\n  \"p50_ttft_s\": " << fmt9(p50_ttft)
     << ",\n  \"p99_ttft_s\": " << fmt9(p99_ttft) << ",\n  \"mean_tpot_s\": " << fmt9(mean_tpot)
     << ",\n  \"mean_queuing_s\": " << fmt9(mean_queuing) << ",\n  \"mean_prefill_s\": " << fmt9(mean_prefill)
     << ",\n  \"queuing_fraction\": " << fmt9(queuing_fraction)
     << ",\n  \"throughput_tokens_per_s\": " << fmt9(throughput_tokens_per_s)
     << ",\n  \"violation_rate\": " << fmt9(violation_rate) << ",\n  \"violations\": " << violations
     << ",\n  \"violations_ttft\": " << violations_ttft << ",\n  \"violations_tpot\": " << violations_tpot
     << ",\n  \"total_output_tokens\": " << total_output_tokens << ",\n  \"makespan_s\": " << fmt9(makespan)
     << ",\n  \"d2h_jobs\": " << d2h_jobs << ",\n  \"d2h_bytes\": " << fmt9(d2h_bytes) << ",\n  \"h2d_jobs\": "
     << h2d_jobs << ",\n  \"h2d_bytes\": " << fmt9(h2d_bytes) << "\n}";
  return os.str();
}

}  // namespace lkv
