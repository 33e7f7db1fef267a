// TEST INFRASTRUCTURE — oracle only. Never linked into the product.
//
// C-ABI shim over the REFERENCE's own C++ classes (compiled in place from
// /root/reference/proj/src by oracle/build_ref.sh into oracle/_ref/). It
// exports the bookkeeping half of include/lkv.h with identical symbols, so
// one Python binding (paper_2410_00428_b200/_abi.py) drives either the
// product or the reference, and parity tests compare them call by call.
//
// The same file is compiled a second time against the PRODUCT headers
// (include/layersim first on the include path) together with the reference
// engine.cpp: that "hybrid" library is the drop-in proof — the reference
// event loop, unmodified, running on the B200 implementation of KvManager,
// PcieBus and the cost model.
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "layersim/engine.hpp"
#include "layersim/errors.hpp"
#include "layersim/workload.hpp"
#include "lkv.h"

using namespace layersim;

struct lkv_kv_manager {
  KvManager impl;
  lkv_kv_manager(BlockPools p, const ModelSpec& m) : impl(p, m) {}
};
struct lkv_pcie_bus {
  PcieBus impl;
  explicit lkv_pcie_bus(double d) : impl(d) {}
};

namespace {
thread_local std::string g_err;

int fail() {
  try {
    throw;
  } catch (const SimulationError& e) {
    g_err = e.what();
    return LKV_ERR_SIMULATION;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return LKV_ERR_CONFIG;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return LKV_ERR_DOMAIN;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return LKV_ERR_INVALID;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LKV_ERR_INTERNAL;
  }
}

ModelSpec M(const lkv_model_spec* m) {
  return {m->n_layers, m->n_heads, m->n_kv_heads, m->d_head, m->hidden, m->n_param, m->f_precision};
}
HardwareSpec H(const lkv_hardware_spec* h) {
  HardwareSpec s;
  s.flops = h->flops;
  s.hbm_bandwidth = h->hbm_bandwidth;
  s.pcie_bandwidth = h->pcie_bandwidth;
  s.nvlink = h->nvlink != 0;
  s.n_gpus = h->n_gpus;
  s.gpu_mem = h->gpu_mem;
  s.kv_reserve_fraction = h->kv_reserve_fraction;
  return s;
}
CostParams P(const lkv_cost_params* c) { return {c->alpha, c->beta, c->gamma, c->delta}; }
OffloadMode mode_of(int32_t m) { return m == LKV_OFFLOAD_HALF ? OffloadMode::Half : OffloadMode::Full; }
}  // namespace

#define TRY try {
#define CATCH      \
  }                \
  catch (...) {    \
    return fail(); \
  }                \
  return LKV_OK;

#ifndef LKV_SHIM_HYBRID
// Reference build: read the private SlotPool::free_stack_ (kv_manager.hpp:
// 153-166) without touching the reference headers. Names in an explicit
// instantiation are exempt from access checking, and the friend each
// instantiation defines returns the member pointer; `auto` avoids naming the
// private types anywhere else.
namespace {
struct GpuPoolTag { friend auto rob(GpuPoolTag); };
struct CpuPoolTag { friend auto rob(CpuPoolTag); };
struct StackTag { friend auto rob(StackTag); };
template <typename Tag, auto P>
struct Rob {
  friend auto rob(Tag) { return P; }
};
template struct Rob<GpuPoolTag, &KvManager::gpu_>;
template struct Rob<CpuPoolTag, &KvManager::cpu_>;
template struct Rob<StackTag, &KvManager::SlotPool::free_stack_>;
}  // namespace
#endif

extern "C" {

const char* lkv_last_error(void) { return g_err.c_str(); }
const char* lkv_version(void) { return "layersim reference shim (oracle)"; }

int lkv_model_validate(const lkv_model_spec* m) { TRY M(m).validate(); CATCH }
int lkv_kv_bytes_per_token_layer(const lkv_model_spec* m, int64_t* o) { TRY *o = kv_bytes_per_token_layer(M(m)); CATCH }
int lkv_prefill_time(const lkv_model_spec* m, const lkv_hardware_spec* h, const lkv_cost_params* c, int64_t s,
                     double* o) { TRY *o = prefill_time(M(m), H(h), P(c), s); CATCH }
int lkv_offload_time(const lkv_model_spec* m, const lkv_hardware_spec* h, const lkv_cost_params* c, int64_t s,
                     int32_t l, double* o) { TRY *o = offload_time(M(m), H(h), P(c), s, l); CATCH }
int lkv_min_retained_layers(const lkv_model_spec* m, const lkv_hardware_spec* h, const lkv_cost_params* c,
                            int64_t s, int32_t* o) { TRY *o = min_retained_layers(M(m), H(h), P(c), s); CATCH }
int lkv_decode_step_time(const lkv_model_spec* m, const lkv_hardware_spec* h, const lkv_cost_params* c,
                         int64_t t, double* o) { TRY *o = decode_step_time(M(m), H(h), P(c), t); CATCH }
int lkv_allreduce_time(const lkv_model_spec* m, const lkv_hardware_spec* h, int64_t t, double* o) {
  TRY *o = allreduce_time(M(m), H(h), t); CATCH
}
int lkv_pool_size_from_hardware(const lkv_model_spec* m, const lkv_hardware_spec* h, const lkv_pool_sizing* s,
                                lkv_block_pools* o) {
  TRY PoolSizing ps;
  ps.max_input_tokens = s->max_input_tokens;
  ps.tokens_per_block = s->tokens_per_block;
  ps.activation_layers_factor = s->activation_layers_factor;
  ps.cpu_pool_multiple = s->cpu_pool_multiple;
  BlockPools p = pool_size_from_hardware(M(m), H(h), ps);
  std::memset(o, 0, sizeof *o);
  o->gpu_blocks_total = p.gpu_blocks_total;
  o->cpu_blocks_total = p.cpu_blocks_total;
  o->tokens_per_block = p.tokens_per_block;
  CATCH
}
int lkv_layer_placement(int32_t L, int32_t x, int32_t* r, int32_t* f) {
  TRY PlacementPlan p = layer_placement(L, x);
  for (std::size_t i = 0; i < p.retained.size(); ++i) if (r) r[i] = p.retained[i];
  for (std::size_t i = 0; i < p.offloaded.size(); ++i) if (f) f[i] = p.offloaded[i];
  CATCH
}

int lkv_kv_create(const lkv_block_pools* p, const lkv_model_spec* m, lkv_kv_manager** o) {
  TRY *o = new lkv_kv_manager({p->gpu_blocks_total, p->cpu_blocks_total, p->tokens_per_block}, M(m)); CATCH
}
int lkv_kv_destroy(lkv_kv_manager* k) { delete k; return LKV_OK; }
int lkv_kv_stats_get(const lkv_kv_manager* k, lkv_kv_stats* o) {
  o->gpu_blocks_total = k->impl.gpu_blocks_total();
  o->gpu_blocks_free = k->impl.gpu_blocks_free();
  o->cpu_blocks_total = k->impl.cpu_blocks_total();
  o->cpu_blocks_free = k->impl.cpu_blocks_free();
  o->tokens_per_block = k->impl.tokens_per_block();
  o->n_layers = 0;
  o->pending_offloads = -1;
  o->live_requests = -1;
  return LKV_OK;
}
int lkv_kv_blocks_per_layer(const lkv_kv_manager* k, int64_t t, int64_t* o) { *o = k->impl.blocks_per_layer(t); return LKV_OK; }
int lkv_kv_request_wise_gpu_blocks(const lkv_kv_manager* k, int64_t t, int64_t* o) {
  *o = k->impl.request_wise_gpu_blocks(t);
  return LKV_OK;
}
int lkv_kv_allocate_prefill(lkv_kv_manager* k, int64_t id, int64_t p, int32_t x, int32_t* ok) {
  TRY *ok = k->impl.allocate_prefill(id, p, x) ? 1 : 0; CATCH
}
int lkv_kv_has_request(const lkv_kv_manager* k, int64_t id, int32_t* o) { *o = k->impl.has_request(id); return LKV_OK; }
int lkv_kv_request_shape(const lkv_kv_manager* k, int64_t id, int64_t* c, int64_t* nb) {
  TRY const RequestKv& r = k->impl.request(id);
  if (c) *c = r.cached_tokens;
  if (nb) *nb = static_cast<int64_t>(r.blocks.size());
  CATCH
}
int lkv_kv_request_table(const lkv_kv_manager* k, int64_t id, lkv_slot_loc* e, int64_t* tb, uint8_t* res) {
  TRY const RequestKv& r = k->impl.request(id);
  const std::size_t L = r.layer_residency.size();
  for (std::size_t b = 0; b < r.blocks.size(); ++b) {
    if (tb) tb[b] = r.blocks[b].token_begin;
    if (!e) continue;
    for (std::size_t l = 0; l < L; ++l) {
      const SlotLoc& s = r.blocks[b].layers[l];
      lkv_slot_loc& o = e[b * L + l];
      o.loc = static_cast<uint8_t>(s.loc);
      o.offload_in_flight = s.offload_in_flight;
      o.pad_ = 0;
      o.slot = s.slot;
      o.dest_slot = s.dest_slot;
    }
  }
  if (res) for (std::size_t l = 0; l < L; ++l) res[l] = static_cast<uint8_t>(r.layer_residency[l]);
  CATCH
}
int lkv_kv_retained_layer_count(const lkv_kv_manager* k, int64_t id, int32_t* o) { TRY *o = k->impl.retained_layer_count(id); CATCH }
int lkv_kv_gpu_blocks_held(const lkv_kv_manager* k, int64_t id, int64_t* o) { TRY *o = k->impl.gpu_blocks_held(id); CATCH }
int lkv_kv_gpu_row_cost(const lkv_kv_manager* k, int64_t id, int64_t* o) { TRY *o = k->impl.gpu_row_cost(id); CATCH }
int lkv_kv_cpu_row_cost(const lkv_kv_manager* k, int64_t id, int64_t* o) { TRY *o = k->impl.cpu_row_cost(id); CATCH }
int lkv_kv_offload_reclaim(const lkv_kv_manager* k, int64_t id, int32_t m, int64_t* o) {
  TRY *o = k->impl.offload_reclaim(id, mode_of(m)); CATCH
}
int lkv_kv_plan_offload(lkv_kv_manager* k, int64_t id, int32_t m, lkv_offload_job* j, int32_t* has) {
  TRY auto r = k->impl.plan_offload(id, mode_of(m));
  std::memset(j, 0, sizeof *j);
  *has = r.has_value();
  if (r) {
    j->job_id = r->job_id;
    j->request_id = r->request_id;
    j->bytes = r->bytes;
    j->layer_count = r->layer_count;
    j->gpu_blocks = r->gpu_blocks;
  }
  CATCH
}
int lkv_kv_complete_offload(lkv_kv_manager* k, int64_t j) { TRY k->impl.complete_offload(j); CATCH }
int lkv_kv_plan_decode_fetch(const lkv_kv_manager* k, int64_t id, lkv_fetch_job* o, int32_t cap, int32_t* n) {
  TRY auto jobs = k->impl.plan_decode_fetch(id);
  *n = static_cast<int32_t>(jobs.size());
  for (int32_t i = 0; i < cap && i < *n; ++i) {
    o[i].layer = jobs[i].layer;
    o[i].pad_ = 0;
    o[i].bytes = jobs[i].bytes;
  }
  CATCH
}
int lkv_kv_needs_append(const lkv_kv_manager* k, int64_t id, int32_t* o) { TRY *o = k->impl.needs_append(id); CATCH }
int lkv_kv_append_decode_block(lkv_kv_manager* k, int64_t id, int32_t* ok) { TRY *ok = k->impl.append_decode_block(id); CATCH }
int lkv_kv_note_token(lkv_kv_manager* k, int64_t id) { TRY k->impl.note_token(id); CATCH }
int lkv_kv_release(lkv_kv_manager* k, int64_t id, lkv_freed_counts* o) {
  TRY auto f = k->impl.release(id);
  if (o) {
    o->gpu = f.gpu;
    o->cpu = f.cpu;
    o->deferred_gpu = f.deferred_gpu;
  }
  CATCH
}
int lkv_kv_check_conservation(const lkv_kv_manager* k) { TRY k->impl.check_conservation(); CATCH }
int lkv_kv_dump_table(const lkv_kv_manager* k, char* buf, size_t cap, size_t* len) {
  TRY std::ostringstream os;
  k->impl.dump_table(os);
  const std::string s = os.str();
  *len = s.size();
  if (buf && cap > s.size()) {
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = 0;
  }
  CATCH
}
#ifdef LKV_SHIM_HYBRID
// hybrid: the product KvManager (its public free_stack)
int lkv_kv_free_stack(const lkv_kv_manager* k, int32_t which, uint32_t* out, int64_t cap, int64_t* size) {
  TRY std::int64_t fresh = 0;
  std::vector<std::uint32_t> pushed;
  k->impl.free_stack(which == 0, &fresh, &pushed);
  const std::int64_t total = which == 0 ? k->impl.gpu_blocks_total() : k->impl.cpu_blocks_total();
  *size = (total - fresh) + static_cast<std::int64_t>(pushed.size());
  if (cap >= *size) {
    for (std::int64_t i = 0; i < total - fresh; ++i) out[i] = static_cast<std::uint32_t>(total - 1 - i);
    std::copy(pushed.begin(), pushed.end(), out + (total - fresh));
  }
  CATCH
}
#else
int lkv_kv_free_stack(const lkv_kv_manager* k, int32_t which, uint32_t* out, int64_t cap, int64_t* size) {
  TRY const auto& pool = which == 0 ? k->impl.*rob(GpuPoolTag{}) : k->impl.*rob(CpuPoolTag{});
  const std::vector<std::uint32_t>& st = pool.*rob(StackTag{});
  *size = static_cast<int64_t>(st.size());
  if (cap >= *size) std::copy(st.begin(), st.end(), out);
  CATCH
}
#endif

#ifdef LKV_SHIM_HYBRID
int lkv_kv_free_delta(lkv_kv_manager* k, int32_t which, int32_t full, int64_t* next_fresh, int64_t* low,
                      int64_t* size, int32_t* changed, uint32_t* out, int64_t cap) {
  TRY const auto d = k->impl.take_free_delta(which == 0, full != 0);
  *next_fresh = d.next_fresh;
  *low = d.low;
  *size = d.size;
  *changed = d.changed ? 1 : 0;
  if (cap >= d.size - d.low) std::copy(d.pushed + d.low, d.pushed + d.size, out);
  CATCH
}
#else
// The reference keeps the whole stack explicitly: every take is a full
// delta with no implicit fresh part (next_fresh = total).
int lkv_kv_free_delta(lkv_kv_manager* k, int32_t which, int32_t, int64_t* next_fresh, int64_t* low, int64_t* size,
                      int32_t* changed, uint32_t* out, int64_t cap) {
  TRY const auto& pool = which == 0 ? k->impl.*rob(GpuPoolTag{}) : k->impl.*rob(CpuPoolTag{});
  const std::vector<std::uint32_t>& st = pool.*rob(StackTag{});
  *next_fresh = which == 0 ? k->impl.gpu_blocks_total() : k->impl.cpu_blocks_total();
  *low = 0;
  *size = static_cast<int64_t>(st.size());
  *changed = 1;
  if (cap >= *size) std::copy(st.begin(), st.end(), out);
  CATCH
}
#endif

int lkv_kv_dump_hash(const lkv_kv_manager* k, uint64_t* o) {
  TRY std::ostringstream os;
  k->impl.dump_table(os);
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : os.str()) {
    h ^= c;
    h *= 1099511628211ull;
  }
  *o = h;
  CATCH
}

int lkv_bus_create(double d, lkv_pcie_bus** o) { TRY *o = new lkv_pcie_bus(d); CATCH }
int lkv_bus_destroy(lkv_pcie_bus* b) { delete b; return LKV_OK; }
int lkv_bus_register_allreduce(lkv_pcie_bus* b, double s, double d, const lkv_hardware_spec* h) {
  TRY b->impl.register_allreduce(s, d, H(h)); CATCH
}
int lkv_bus_submit_transfer(lkv_pcie_bus* b, double bytes, int32_t dir, double t, double chunk,
                            const lkv_hardware_spec* h, lkv_transfer_schedule* o) {
  TRY TransferSchedule s = b->impl.submit_transfer(
      {bytes, dir == LKV_D2H ? Direction::DeviceToHost : Direction::HostToDevice, t, chunk}, H(h));
  o->start = s.start;
  o->completion = s.completion;
  o->chunks = s.chunks;
  o->deferrals = s.deferrals;
  CATCH
}
int lkv_bus_state(const lkv_pcie_bus* b, double t, double* bu, double* ab, int32_t* a) {
  if (bu) *bu = b->impl.busy_until();
  if (ab) *ab = b->impl.allreduce_busy_until();
  if (a) *a = b->impl.allreduce_active(t);
  return LKV_OK;
}
int lkv_bus_enable_history(lkv_pcie_bus* b, int32_t on) { b->impl.enable_history(on != 0); return LKV_OK; }
static int spans(const std::vector<PcieBus::Span>& v, lkv_span* o, int32_t cap, int32_t* n) {
  *n = static_cast<int32_t>(v.size());
  for (int32_t i = 0; i < cap && i < *n; ++i) {
    o[i].begin = v[i].begin;
    o[i].end = v[i].end;
    o[i].is_allreduce = v[i].is_allreduce;
    o[i].pad_ = 0;
  }
  return LKV_OK;
}
int lkv_bus_chunk_history(const lkv_pcie_bus* b, lkv_span* o, int32_t cap, int32_t* n) {
  return spans(b->impl.chunk_history(), o, cap, n);
}
int lkv_bus_allreduce_windows(const lkv_pcie_bus* b, lkv_span* o, int32_t cap, int32_t* n) {
  return spans(b->impl.allreduce_windows(), o, cap, n);
}
int lkv_schedule_prefill_span(const lkv_model_spec* m, const lkv_hardware_spec* h, const lkv_cost_params* c,
                              lkv_pcie_bus* bus, const int32_t* off, int32_t n_off, int64_t prompt, double start,
                              double chunk, int32_t enabled, double* comp, lkv_transfer_schedule* jobs,
                              int32_t cap, int32_t* n_jobs) {
  TRY std::vector<int> o(off, off + n_off);
  PrefillSchedule s = schedule_prefill_span(M(m), H(h), P(c), bus->impl, o, prompt, start, chunk, enabled != 0);
  *comp = s.completion;
  *n_jobs = static_cast<int32_t>(s.jobs.size());
  for (int32_t i = 0; i < cap && i < *n_jobs; ++i) {
    jobs[i].start = s.jobs[i].start;
    jobs[i].completion = s.jobs[i].completion;
    jobs[i].chunks = s.jobs[i].chunks;
    jobs[i].deferrals = s.jobs[i].deferrals;
  }
  CATCH
}

// ---- full engine run (reference Engine::run, engine.cpp:76-121) ----------------
typedef struct ref_engine_cfg {
  lkv_model_spec model;
  lkv_hardware_spec hw;
  lkv_cost_params cost;
  double ttft_slo, tpot_slo;
  int32_t policy_layerkv, slo_scheduler;
  int64_t gpu_blocks, cpu_blocks;
  int32_t tokens_per_block, horizon;
  double threshold_fraction, predictor_accuracy;
  int64_t max_batch_tokens;
  double max_sim_time, chunk_bytes;
  uint64_t seed;
  int32_t force_retained_layers, invariant_checks;
} ref_engine_cfg;

typedef struct ref_engine_out {
  double mean_ttft, p50_ttft, p99_ttft, mean_tpot, throughput, makespan;
  int64_t d2h_jobs, h2d_jobs;
  double d2h_bytes, h2d_bytes;
  int32_t completed, n_rows;
} ref_engine_out;

// Trace given as arrays (id, arrival, prompt, output). requests.csv text is
// written to csv (when cap suffices); *csv_len = its length.
static EngineConfig engine_cfg(const ref_engine_cfg* c) {
  EngineConfig e;
  e.model = M(&c->model);
  e.hw = H(&c->hw);
  e.cost = P(&c->cost);
  e.slo.ttft_slo = c->ttft_slo;
  e.slo.tpot_slo = c->tpot_slo;
  e.policy.kind = c->policy_layerkv ? PolicyKind::LayerKv : PolicyKind::BaselineRequestWise;
  e.policy.slo_scheduler_enabled = c->slo_scheduler != 0;
  e.pools = {c->gpu_blocks, c->cpu_blocks, c->tokens_per_block};
  e.scheduler.threshold_fraction = c->threshold_fraction;
  e.scheduler.horizon = c->horizon;
  e.scheduler.predictor_accuracy = c->predictor_accuracy;
  e.max_batch_tokens = c->max_batch_tokens;
  e.max_sim_time = c->max_sim_time;
  e.chunk_bytes = c->chunk_bytes;
  e.seed = c->seed;
  e.force_retained_layers = c->force_retained_layers;
  e.invariant_checks = c->invariant_checks != 0;
  e.keep_transfer_log = true;
  e.keep_decision_log = true;
  return e;
}

static Trace engine_trace(const ref_engine_cfg* c, int32_t n, const int64_t* ids, const double* arrival,
                          const int32_t* prompt, const int32_t* output) {
  Trace t;
  t.seed = c->seed;
  for (int32_t i = 0; i < n; ++i) t.requests.push_back({ids[i], arrival[i], prompt[i], output[i]});
  return t;
}

LKV_API int ref_engine_run(const ref_engine_cfg* c, int32_t n, const int64_t* ids, const double* arrival,
                   const int32_t* prompt, const int32_t* output, ref_engine_out* out, char* csv,
                   size_t cap, size_t* csv_len) {
  TRY Engine eng(engine_cfg(c), engine_trace(c, n, ids, arrival, prompt, output));
  MetricsReport r = eng.run();
  std::memset(out, 0, sizeof *out);
  out->mean_ttft = r.mean_ttft;
  out->p50_ttft = r.p50_ttft;
  out->p99_ttft = r.p99_ttft;
  out->mean_tpot = r.mean_tpot;
  out->throughput = r.throughput_tokens_per_s;
  out->makespan = r.makespan;
  out->completed = r.completed;
  out->n_rows = static_cast<int32_t>(r.per_request.size());
  for (const auto& row : eng.transfer_log()) {
    if (row.direction == Direction::DeviceToHost) {
      ++out->d2h_jobs;
      out->d2h_bytes += row.bytes;
    } else {
      ++out->h2d_jobs;
      out->h2d_bytes += row.bytes;
    }
  }
  const std::string s = r.requests_csv();
  *csv_len = s.size();
  if (csv && cap > s.size()) {
    std::memcpy(csv, s.data(), s.size());
    csv[s.size()] = 0;
  }
  CATCH
}

// transfer_log.csv (which = 0) or decision_log.csv (which = 1) of the same
// run, as the reference CLI writes them (tools/layersim_main.cpp:96-117: the
// CLI itself needs the absent CLI11, so its few formatting lines are restated
// here over Engine::transfer_log() / decision_log()).
LKV_API int ref_engine_log(const ref_engine_cfg* c, int32_t n, const int64_t* ids, const double* arrival,
                   const int32_t* prompt, const int32_t* output, int32_t which, char* buf, size_t cap,
                   size_t* len) {
  TRY Engine eng(engine_cfg(c), engine_trace(c, n, ids, arrival, prompt, output));
  eng.run();
  std::ostringstream os;
  if (which == 0) {
    os << "submit_s,start_s,end_s,bytes,direction,deferrals\n";
    for (const auto& row : eng.transfer_log()) {
      os << format_double(row.submit) << ',' << format_double(row.start) << ',' << format_double(row.end) << ','
         << format_double(row.bytes) << ',' << (row.direction == Direction::DeviceToHost ? "d2h" : "h2d") << ','
         << row.deferrals << "\n";
    }
  } else {
    os << "time_s,min_budget_s,admitted,offload_plan\n";
    for (const auto& row : eng.decision_log()) {
      const char* plan = row.plan == OffloadPlanKind::None ? "none" : (row.plan == OffloadPlanKind::Half ? "half" : "full");
      os << format_double(row.time) << ',' << format_double(row.min_budget) << ',' << row.admitted << ',' << plan
         << "\n";
    }
  }
  const std::string s = os.str();
  *len = s.size();
  if (buf && cap > s.size()) {
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = 0;
  }
  CATCH
}

// Reference trace generators (workload.cpp:34-82): writes up to cap requests.
LKV_API int ref_generate_trace(int32_t kind_sharegpt, int32_t n, int32_t prompt, int32_t output, double rate,
                       uint64_t seed, int64_t* ids, double* arrival, int32_t* p, int32_t* o) {
  TRY Trace t = kind_sharegpt ? generate_sharegpt_like(n, rate, seed) : generate_fixed(n, prompt, output, rate, seed);
  for (std::size_t i = 0; i < t.requests.size(); ++i) {
    ids[i] = t.requests[i].id;
    arrival[i] = t.requests[i].arrival;
    p[i] = t.requests[i].prompt_tokens;
    o[i] = t.requests[i].output_tokens;
  }
  CATCH
}

// Reference load_trace / save_trace (workload.cpp:84-148): JSONL format parity.
// Returns the record count (arrays filled up to cap), or -1 on error.
LKV_API int ref_load_trace(const char* path, int64_t* ids, double* arrival, int32_t* p, int32_t* o, int32_t cap) {
  try {
    Trace t = load_trace(path);
    for (std::size_t i = 0; i < t.requests.size() && static_cast<int32_t>(i) < cap; ++i) {
      ids[i] = t.requests[i].id;
      arrival[i] = t.requests[i].arrival;
      p[i] = t.requests[i].prompt_tokens;
      o[i] = t.requests[i].output_tokens;
    }
    return static_cast<int>(t.requests.size());
  } catch (...) {
    return -1;
  }
}

LKV_API int ref_save_trace(const char* path, int32_t n, const int64_t* ids, const double* arrival, const int32_t* p,
                           const int32_t* o) {
  TRY Trace t;
  for (int32_t i = 0; i < n; ++i) t.requests.push_back({ids[i], arrival[i], p[i], o[i]});
  save_trace(t, path);
  CATCH
}

}  // extern "C"
