// extern "C" bookkeeping half of include/lkv.h: converts between the plain C
// structs and the C++ drop-in classes, and exceptions into status codes.
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>

#include "layersim/errors.hpp"
#include "layersim/interconnect.hpp"
#include "layersim/kv_manager.hpp"
#include "layersim/prefill_span.hpp"
#include "lkv.h"
#include "lkv_internal.hpp"

using namespace layersim;

struct lkv_kv_manager {
  KvManager impl;
  lkv_kv_manager(BlockPools p, const ModelSpec& m) : impl(p, m) {}
};

struct lkv_pcie_bus {
  PcieBus impl;
  explicit lkv_pcie_bus(double d) : impl(d) {}
};

namespace lkv {

namespace {
thread_local std::string g_error;
}

void set_error(const std::string& msg) { g_error = msg; }

int status_from_current_exception() {
  try {
    throw;
  } catch (const SimulationError& e) {
    g_error = e.what();
    return LKV_ERR_SIMULATION;
  } catch (const ConfigError& e) {
    g_error = e.what();
    return LKV_ERR_CONFIG;
  } catch (const CapacityError& e) {
    g_error = e.what();
    return LKV_ERR_CAPACITY;
  } catch (const CudaError& e) {
    g_error = e.what();
    return LKV_ERR_CUDA;
  } catch (const std::domain_error& e) {
    g_error = e.what();
    return LKV_ERR_DOMAIN;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return LKV_ERR_INVALID;
  } catch (const std::length_error& e) {  // a bounded arena (e.g. pinned host frames) is exhausted
    g_error = e.what();
    return LKV_ERR_CAPACITY;
  } catch (const std::exception& e) {
    g_error = e.what();
    return LKV_ERR_INTERNAL;
  } catch (...) {
    g_error = "unknown exception";
    return LKV_ERR_INTERNAL;
  }
}

ModelSpec to_model(const lkv_model_spec* m) {
  ModelSpec s;
  s.n_layers = m->n_layers;
  s.n_heads = m->n_heads;
  s.n_kv_heads = m->n_kv_heads;
  s.d_head = m->d_head;
  s.hidden = m->hidden;
  s.n_param = m->n_param;
  s.f_precision = m->f_precision;
  return s;
}

HardwareSpec to_hw(const lkv_hardware_spec* h) {
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

CostParams to_cost(const lkv_cost_params* c) {
  CostParams p;
  p.alpha = c->alpha;
  p.beta = c->beta;
  p.gamma = c->gamma;
  p.delta = c->delta;
  return p;
}

KvManager& kv_impl(lkv_kv_manager* kv) { return kv->impl; }

}  // namespace lkv

using lkv::status_from_current_exception;

#define LKV_TRY try {
#define LKV_CATCH                           \
  }                                         \
  catch (...) {                             \
    return status_from_current_exception(); \
  }                                         \
  return LKV_OK;
#define LKV_REQUIRE(cond)                                     \
  do {                                                        \
    if (!(cond)) {                                            \
      lkv::set_error("invalid argument: " #cond);             \
      return LKV_ERR_INVALID;                                 \
    }                                                         \
  } while (0)

extern "C" {

const char* lkv_last_error(void) { return lkv::g_error.c_str(); }
const char* lkv_version(void) { return "lkv 0.1.0 sm_100a"; }

// ---- cost model -------------------------------------------------------------
int lkv_model_validate(const lkv_model_spec* m) {
  LKV_REQUIRE(m);
  LKV_TRY lkv::to_model(m).validate();
  LKV_CATCH
}

int lkv_kv_bytes_per_token_layer(const lkv_model_spec* m, int64_t* out) {
  LKV_REQUIRE(m && out);
  LKV_TRY* out = kv_bytes_per_token_layer(lkv::to_model(m));
  LKV_CATCH
}

int lkv_prefill_time(const lkv_model_spec* m, const lkv_hardware_spec* h,
                     const lkv_cost_params* c, int64_t seqlen, double* out) {
  LKV_REQUIRE(m && h && c && out);
  LKV_TRY* out = prefill_time(lkv::to_model(m), lkv::to_hw(h), lkv::to_cost(c), seqlen);
  LKV_CATCH
}

int lkv_offload_time(const lkv_model_spec* m, const lkv_hardware_spec* h,
                     const lkv_cost_params* c, int64_t seqlen, int32_t layers, double* out) {
  LKV_REQUIRE(m && h && c && out);
  LKV_TRY* out = offload_time(lkv::to_model(m), lkv::to_hw(h), lkv::to_cost(c), seqlen, layers);
  LKV_CATCH
}

int lkv_min_retained_layers(const lkv_model_spec* m, const lkv_hardware_spec* h,
                            const lkv_cost_params* c, int64_t seqlen, int32_t* out) {
  LKV_REQUIRE(m && h && c && out);
  LKV_TRY* out = min_retained_layers(lkv::to_model(m), lkv::to_hw(h), lkv::to_cost(c), seqlen);
  LKV_CATCH
}

int lkv_decode_step_time(const lkv_model_spec* m, const lkv_hardware_spec* h,
                         const lkv_cost_params* c, int64_t tokens, double* out) {
  LKV_REQUIRE(m && h && c && out);
  LKV_TRY* out = decode_step_time(lkv::to_model(m), lkv::to_hw(h), lkv::to_cost(c), tokens);
  LKV_CATCH
}

int lkv_allreduce_time(const lkv_model_spec* m, const lkv_hardware_spec* h, int64_t tokens,
                       double* out) {
  LKV_REQUIRE(m && h && out);
  LKV_TRY* out = allreduce_time(lkv::to_model(m), lkv::to_hw(h), tokens);
  LKV_CATCH
}

// ---- sizing / placement -----------------------------------------------------
int lkv_pool_size_from_hardware(const lkv_model_spec* m, const lkv_hardware_spec* h,
                                const lkv_pool_sizing* s, lkv_block_pools* out) {
  LKV_REQUIRE(m && h && s && out);
  LKV_TRY PoolSizing ps;
  ps.max_input_tokens = s->max_input_tokens;
  ps.tokens_per_block = s->tokens_per_block;
  ps.activation_layers_factor = s->activation_layers_factor;
  ps.cpu_pool_multiple = s->cpu_pool_multiple;
  BlockPools p = pool_size_from_hardware(lkv::to_model(m), lkv::to_hw(h), ps);
  std::memset(out, 0, sizeof *out);
  out->gpu_blocks_total = p.gpu_blocks_total;
  out->cpu_blocks_total = p.cpu_blocks_total;
  out->tokens_per_block = p.tokens_per_block;
  LKV_CATCH
}

int lkv_layer_placement(int32_t n_layers, int32_t x, int32_t* retained, int32_t* offloaded) {
  LKV_TRY PlacementPlan p = layer_placement(n_layers, x);
  for (std::size_t i = 0; i < p.retained.size(); ++i)
    if (retained) retained[i] = p.retained[i];
  for (std::size_t i = 0; i < p.offloaded.size(); ++i)
    if (offloaded) offloaded[i] = p.offloaded[i];
  LKV_CATCH
}

// ---- KvManager ----------------------------------------------------------------
int lkv_kv_create(const lkv_block_pools* pools, const lkv_model_spec* m, lkv_kv_manager** out) {
  LKV_REQUIRE(pools && m && out);
  LKV_TRY BlockPools p;
  p.gpu_blocks_total = pools->gpu_blocks_total;
  p.cpu_blocks_total = pools->cpu_blocks_total;
  p.tokens_per_block = pools->tokens_per_block;
  if (p.tokens_per_block <= 0 || p.gpu_blocks_total < 0 || p.cpu_blocks_total < 0 ||
      p.gpu_blocks_total > 0xFFFFFFFFll || p.cpu_blocks_total > 0xFFFFFFFFll) {
    throw std::invalid_argument("lkv_kv_create: pool sizes must fit uint32 slots");
  }
  *out = new lkv_kv_manager(p, lkv::to_model(m));
  LKV_CATCH
}

int lkv_kv_destroy(lkv_kv_manager* kv) {
  delete kv;
  return LKV_OK;
}

int lkv_kv_stats_get(const lkv_kv_manager* kv, lkv_kv_stats* out) {
  LKV_REQUIRE(kv && out);
  const KvManager& k = kv->impl;
  out->gpu_blocks_total = k.gpu_blocks_total();
  out->gpu_blocks_free = k.gpu_blocks_free();
  out->cpu_blocks_total = k.cpu_blocks_total();
  out->cpu_blocks_free = k.cpu_blocks_free();
  out->tokens_per_block = k.tokens_per_block();
  out->n_layers = k.n_layers();
  out->pending_offloads = k.pending_offload_count();
  out->live_requests = static_cast<int64_t>(k.request_ids().size());
  return LKV_OK;
}

int lkv_kv_blocks_per_layer(const lkv_kv_manager* kv, int64_t tokens, int64_t* out) {
  LKV_REQUIRE(kv && out);
  *out = kv->impl.blocks_per_layer(tokens);
  return LKV_OK;
}

int lkv_kv_request_wise_gpu_blocks(const lkv_kv_manager* kv, int64_t prompt, int64_t* out) {
  LKV_REQUIRE(kv && out);
  *out = kv->impl.request_wise_gpu_blocks(prompt);
  return LKV_OK;
}

int lkv_kv_allocate_prefill(lkv_kv_manager* kv, int64_t id, int64_t prompt, int32_t x,
                            int32_t* ok) {
  LKV_REQUIRE(kv && ok);
  LKV_TRY* ok = kv->impl.allocate_prefill(id, prompt, x) ? 1 : 0;
  LKV_CATCH
}

int lkv_kv_has_request(const lkv_kv_manager* kv, int64_t id, int32_t* out) {
  LKV_REQUIRE(kv && out);
  *out = kv->impl.has_request(id) ? 1 : 0;
  return LKV_OK;
}

int lkv_kv_request_shape(const lkv_kv_manager* kv, int64_t id, int64_t* cached, int64_t* nb) {
  LKV_REQUIRE(kv);
  LKV_TRY const RequestKv& r = kv->impl.request(id);
  if (cached) *cached = r.cached_tokens;
  if (nb) *nb = static_cast<int64_t>(r.blocks.size());
  LKV_CATCH
}

int lkv_kv_request_table(const lkv_kv_manager* kv, int64_t id, lkv_slot_loc* entries,
                         int64_t* token_begin, uint8_t* residency) {
  LKV_REQUIRE(kv);
  LKV_TRY const RequestKv& r = kv->impl.request(id);
  const int L = kv->impl.n_layers();
  for (std::size_t b = 0; b < r.blocks.size(); ++b) {
    if (token_begin) token_begin[b] = r.blocks[b].token_begin;
    if (!entries) continue;
    for (int l = 0; l < L; ++l) {
      const SlotLoc& e = r.blocks[b].layers[static_cast<std::size_t>(l)];
      lkv_slot_loc& o = entries[b * static_cast<std::size_t>(L) + static_cast<std::size_t>(l)];
      o.loc = static_cast<uint8_t>(e.loc);
      o.offload_in_flight = e.offload_in_flight ? 1 : 0;
      o.pad_ = 0;
      o.slot = e.slot;
      o.dest_slot = e.dest_slot;
    }
  }
  if (residency)
    for (int l = 0; l < L; ++l)
      residency[l] = static_cast<uint8_t>(r.layer_residency[static_cast<std::size_t>(l)]);
  LKV_CATCH
}

int lkv_kv_retained_layer_count(const lkv_kv_manager* kv, int64_t id, int32_t* out) {
  LKV_REQUIRE(kv && out);
  LKV_TRY* out = kv->impl.retained_layer_count(id);
  LKV_CATCH
}

int lkv_kv_gpu_blocks_held(const lkv_kv_manager* kv, int64_t id, int64_t* out) {
  LKV_REQUIRE(kv && out);
  LKV_TRY* out = kv->impl.gpu_blocks_held(id);
  LKV_CATCH
}

int lkv_kv_gpu_row_cost(const lkv_kv_manager* kv, int64_t id, int64_t* out) {
  LKV_REQUIRE(kv && out);
  LKV_TRY* out = kv->impl.gpu_row_cost(id);
  LKV_CATCH
}

int lkv_kv_cpu_row_cost(const lkv_kv_manager* kv, int64_t id, int64_t* out) {
  LKV_REQUIRE(kv && out);
  LKV_TRY* out = kv->impl.cpu_row_cost(id);
  LKV_CATCH
}

int lkv_kv_offload_reclaim(const lkv_kv_manager* kv, int64_t id, int32_t mode, int64_t* out) {
  LKV_REQUIRE(kv && out && (mode == LKV_OFFLOAD_HALF || mode == LKV_OFFLOAD_FULL));
  LKV_TRY* out =
      kv->impl.offload_reclaim(id, mode == LKV_OFFLOAD_HALF ? OffloadMode::Half : OffloadMode::Full);
  LKV_CATCH
}

int lkv_kv_plan_offload(lkv_kv_manager* kv, int64_t id, int32_t mode, lkv_offload_job* job,
                        int32_t* has_value) {
  LKV_REQUIRE(kv && job && has_value && (mode == LKV_OFFLOAD_HALF || mode == LKV_OFFLOAD_FULL));
  LKV_TRY auto j =
      kv->impl.plan_offload(id, mode == LKV_OFFLOAD_HALF ? OffloadMode::Half : OffloadMode::Full);
  std::memset(job, 0, sizeof *job);
  *has_value = j.has_value() ? 1 : 0;
  if (j) {
    job->job_id = j->job_id;
    job->request_id = j->request_id;
    job->bytes = j->bytes;
    job->layer_count = j->layer_count;
    job->gpu_blocks = j->gpu_blocks;
  }
  LKV_CATCH
}

int lkv_kv_complete_offload(lkv_kv_manager* kv, int64_t job_id) {
  LKV_REQUIRE(kv);
  LKV_TRY kv->impl.complete_offload(job_id);
  LKV_CATCH
}

int lkv_kv_plan_decode_fetch(const lkv_kv_manager* kv, int64_t id, lkv_fetch_job* out,
                             int32_t cap, int32_t* count) {
  LKV_REQUIRE(kv && count && cap >= 0);
  LKV_TRY std::vector<FetchJob> jobs = kv->impl.plan_decode_fetch(id);
  *count = static_cast<int32_t>(jobs.size());
  for (int32_t i = 0; i < cap && i < *count; ++i) {
    out[i].layer = jobs[static_cast<std::size_t>(i)].layer;
    out[i].pad_ = 0;
    out[i].bytes = jobs[static_cast<std::size_t>(i)].bytes;
  }
  LKV_CATCH
}

int lkv_kv_needs_append(const lkv_kv_manager* kv, int64_t id, int32_t* out) {
  LKV_REQUIRE(kv && out);
  LKV_TRY* out = kv->impl.needs_append(id) ? 1 : 0;
  LKV_CATCH
}

int lkv_kv_append_decode_block(lkv_kv_manager* kv, int64_t id, int32_t* ok) {
  LKV_REQUIRE(kv && ok);
  LKV_TRY* ok = kv->impl.append_decode_block(id) ? 1 : 0;
  LKV_CATCH
}

int lkv_kv_note_token(lkv_kv_manager* kv, int64_t id) {
  LKV_REQUIRE(kv);
  LKV_TRY kv->impl.note_token(id);
  LKV_CATCH
}

int lkv_kv_release(lkv_kv_manager* kv, int64_t id, lkv_freed_counts* out) {
  LKV_REQUIRE(kv);
  LKV_TRY KvManager::FreedCounts f = kv->impl.release(id);
  if (out) {
    out->gpu = f.gpu;
    out->cpu = f.cpu;
    out->deferred_gpu = f.deferred_gpu;
  }
  LKV_CATCH
}

int lkv_kv_check_conservation(const lkv_kv_manager* kv) {
  LKV_REQUIRE(kv);
  LKV_TRY kv->impl.check_conservation();
  LKV_CATCH
}

int lkv_kv_dump_table(const lkv_kv_manager* kv, char* buf, size_t cap, size_t* len) {
  LKV_REQUIRE(kv && len);
  LKV_TRY std::ostringstream os;
  kv->impl.dump_table(os);
  const std::string s = os.str();
  *len = s.size();
  if (buf && cap > s.size()) {
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = '\0';
  }
  LKV_CATCH
}

int lkv_kv_free_stack(const lkv_kv_manager* kv, int32_t which, uint32_t* out, int64_t cap, int64_t* size) {
  LKV_REQUIRE(kv && (which == 0 || which == 1) && size && (out || cap == 0));
  LKV_TRY std::int64_t fresh = 0;
  std::vector<std::uint32_t> pushed;
  kv->impl.free_stack(which == 0, &fresh, &pushed);
  const std::int64_t total = which == 0 ? kv->impl.gpu_blocks_total() : kv->impl.cpu_blocks_total();
  *size = (total - fresh) + static_cast<std::int64_t>(pushed.size());
  if (cap >= *size) {
    for (std::int64_t i = 0; i < total - fresh; ++i) out[i] = static_cast<std::uint32_t>(total - 1 - i);
    std::copy(pushed.begin(), pushed.end(), out + (total - fresh));
  }
  LKV_CATCH
}

int lkv_kv_free_delta(lkv_kv_manager* kv, int32_t which, int32_t full, int64_t* next_fresh, int64_t* low,
                      int64_t* size, int32_t* changed, uint32_t* out, int64_t cap) {
  LKV_REQUIRE(kv && (which == 0 || which == 1) && next_fresh && low && size && changed && (out || cap == 0));
  LKV_TRY const auto d = kv->impl.take_free_delta(which == 0, full != 0);
  *next_fresh = d.next_fresh;
  *low = d.low;
  *size = d.size;
  *changed = d.changed ? 1 : 0;
  if (cap >= d.size - d.low) std::copy(d.pushed + d.low, d.pushed + d.size, out);
  LKV_CATCH
}

int lkv_kv_dump_hash(const lkv_kv_manager* kv, uint64_t* out) {
  LKV_REQUIRE(kv && out);
  LKV_TRY std::ostringstream os;
  kv->impl.dump_table(os);
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : os.str()) {
    h ^= c;
    h *= 1099511628211ull;
  }
  *out = h;
  LKV_CATCH
}

// ---- PcieBus ------------------------------------------------------------------
int lkv_bus_create(double delta, lkv_pcie_bus** out) {
  LKV_REQUIRE(out);
  LKV_TRY* out = new lkv_pcie_bus(delta);
  LKV_CATCH
}

int lkv_bus_destroy(lkv_pcie_bus* bus) {
  delete bus;
  return LKV_OK;
}

int lkv_bus_register_allreduce(lkv_pcie_bus* bus, double start, double dur,
                               const lkv_hardware_spec* hw) {
  LKV_REQUIRE(bus && hw);
  LKV_TRY bus->impl.register_allreduce(start, dur, lkv::to_hw(hw));
  LKV_CATCH
}

int lkv_bus_submit_transfer(lkv_pcie_bus* bus, double bytes, int32_t dir, double submit,
                            double chunk, const lkv_hardware_spec* hw,
                            lkv_transfer_schedule* out) {
  LKV_REQUIRE(bus && hw && out && (dir == LKV_D2H || dir == LKV_H2D));
  LKV_TRY TransferJob j;
  j.bytes = bytes;
  j.direction = dir == LKV_D2H ? Direction::DeviceToHost : Direction::HostToDevice;
  j.submit_time = submit;
  j.chunk_bytes = chunk;
  TransferSchedule s = bus->impl.submit_transfer(j, lkv::to_hw(hw));
  out->start = s.start;
  out->completion = s.completion;
  out->chunks = s.chunks;
  out->deferrals = s.deferrals;
  LKV_CATCH
}

int lkv_bus_state(const lkv_pcie_bus* bus, double t, double* busy, double* ar_busy,
                  int32_t* active) {
  LKV_REQUIRE(bus);
  if (busy) *busy = bus->impl.busy_until();
  if (ar_busy) *ar_busy = bus->impl.allreduce_busy_until();
  if (active) *active = bus->impl.allreduce_active(t) ? 1 : 0;
  return LKV_OK;
}

int lkv_bus_enable_history(lkv_pcie_bus* bus, int32_t on) {
  LKV_REQUIRE(bus);
  bus->impl.enable_history(on != 0);
  return LKV_OK;
}

static int copy_spans(const std::vector<PcieBus::Span>& v, lkv_span* out, int32_t cap,
                      int32_t* count) {
  *count = static_cast<int32_t>(v.size());
  for (int32_t i = 0; i < cap && i < *count; ++i) {
    out[i].begin = v[static_cast<std::size_t>(i)].begin;
    out[i].end = v[static_cast<std::size_t>(i)].end;
    out[i].is_allreduce = v[static_cast<std::size_t>(i)].is_allreduce ? 1 : 0;
    out[i].pad_ = 0;
  }
  return LKV_OK;
}

int lkv_bus_chunk_history(const lkv_pcie_bus* bus, lkv_span* out, int32_t cap, int32_t* count) {
  LKV_REQUIRE(bus && count && cap >= 0);
  return copy_spans(bus->impl.chunk_history(), out, cap, count);
}

int lkv_bus_allreduce_windows(const lkv_pcie_bus* bus, lkv_span* out, int32_t cap,
                              int32_t* count) {
  LKV_REQUIRE(bus && count && cap >= 0);
  return copy_spans(bus->impl.allreduce_windows(), out, cap, count);
}

int lkv_schedule_prefill_span(const lkv_model_spec* m, const lkv_hardware_spec* h,
                              const lkv_cost_params* c, lkv_pcie_bus* bus,
                              const int32_t* offloaded, int32_t n_off, int64_t prompt,
                              double start, double chunk, int32_t enabled, double* completion,
                              lkv_transfer_schedule* jobs, int32_t cap, int32_t* n_jobs) {
  LKV_REQUIRE(m && h && c && bus && completion && n_jobs && n_off >= 0 && cap >= 0);
  LKV_TRY std::vector<int> off(offloaded, offloaded + n_off);
  PrefillSchedule s = schedule_prefill_span(lkv::to_model(m), lkv::to_hw(h), lkv::to_cost(c),
                                            bus->impl, off, prompt, start, chunk, enabled != 0);
  *completion = s.completion;
  *n_jobs = static_cast<int32_t>(s.jobs.size());
  for (int32_t i = 0; i < cap && i < *n_jobs; ++i) {
    const TransferSchedule& t = s.jobs[static_cast<std::size_t>(i)];
    jobs[i].start = t.start;
    jobs[i].completion = t.completion;
    jobs[i].chunks = t.chunks;
    jobs[i].deferrals = t.deferrals;
  }
  LKV_CATCH
}

}  // extern "C"
