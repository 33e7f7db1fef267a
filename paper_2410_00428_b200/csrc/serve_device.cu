// Device executor of the serving loop and the serving /
// trace C ABI (include/lkv.h, "serving loop" section).
//
// Every piece of work the loop schedules runs on the GPU through the data
// path (lkv_device):
//   prefill of a request: per layer, the generator K/V (stand-in for the K/V
//     projection output), the layer's dense GEMMs (cuBLAS bf16, random
//     weights; plain library GEMMs), the tcgen05 causal prefill attention,
//     then lkv_prefill_layer — scatter into GPU slots or pack + D2H into the
//     CPU slots' pinned frames on the copy engine, overlapped with the next
//     layer (engine.cpp:27-42 models exactly this span);
//   escalation: kv.plan_offload itself starts the gather + D2H (observer);
//   decode iteration: lkv_decode_begin_append, then per layer the new
//     tokens' generator K/V, the dense GEMMs (M = batch), the write-back of
//     the new token (f2) and the paged attention after the layer's prefetch
//     (engine.cpp:405-453 models this pipeline).
// Clock "virtual": times still come from the cost model + PcieBus (the same
// ModelledExecutor the modelled loop uses), so the run reproduces the
// reference's requests.csv while the device really moves every byte; with
// verify_kv every request's KV is checked bit-exact against the generator
// right before release. Clock "measured": CUDA events give the times.
#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <deque>
#include <limits>
#include <stdexcept>
#include <string>

#include "layersim/errors.hpp"
#include "lkv.h"
#include "lkv/serve.hpp"
#include "lkv_internal.hpp"

namespace lkv {
cudaEvent_t device_job_event(lkv_device* d, std::int64_t job_id);  // device.cu
}

namespace {

using lkv::CudaError;

#define SERVE_CUDA(expr)                                                                              \
  do {                                                                                                \
    cudaError_t e_ = (expr);                                                                          \
    if (e_ != cudaSuccess)                                                                            \
      throw CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_) + " (serve_device.cu:" +     \
                      std::to_string(__LINE__) + ")");                                                \
  } while (0)
#define SERVE_BLAS(expr)                                                                              \
  do {                                                                                                \
    cublasStatus_t s_ = (expr);                                                                       \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                                  \
      throw CudaError(std::string(#expr) + ": cublas status " + std::to_string(static_cast<int>(s_))); \
  } while (0)
#define SERVE_LKV(expr)                                                  \
  do {                                                                   \
    if ((expr) != LKV_OK) throw CudaError(std::string(#expr) + ": " + lkv_last_error()); \
  } while (0)

__global__ void fill_uniform_bf16(__nv_bfloat16* p, long long n, unsigned long long seed, float scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = seed + (static_cast<unsigned long long>(i) + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    const float u = static_cast<float>(z >> 40) * (1.0f / 16777216.0f) - 0.5f;
    p[i] = __float2bfloat16_rn(u * scale);
  }
}

struct DeviceOptions {
  bool measured = false;
  bool dense = true;
  bool attention = true;
  bool verify = false;
  int device = 0;
  int depth = 2;
  std::int64_t ffn = 0;
  std::int64_t host_slots = 0;
  std::uint64_t kv_seed = 0x4C61796572ull;
  int tp_rank = 0;
  std::int64_t pinned_frames = 0;  // > 0: tiered host memory (f3)
};

struct TraceShape {
  std::int64_t max_prompt = 1, max_total = 1;
  std::int64_t all_blocks = 1;  // sum over requests of blocks per layer at completion (+1 headroom)
  int n = 1;
};

class DeviceExecutor final : public lkv::Executor {
 public:
  DeviceExecutor(const lkv::ServeConfig& cfg, layersim::KvManager& kv, const DeviceOptions& o, const TraceShape& tr)
      : cfg_(cfg), kv_(kv), o_(o), modelled_(cfg, kv) {
    const auto& m = cfg.model;
    const int bs = cfg.pools.tokens_per_block;
    lkv_model_spec ms{m.n_layers, m.n_heads, m.n_kv_heads, m.d_head, m.hidden, m.n_param, m.f_precision, 0};
    lkv_device_config dc{};
    dc.device = o.device;
    dc.tp_rank = o.tp_rank;  // one KV-head shard of hw.n_gpus (the slot ids are the same on every rank)
    dc.tp_size = cfg.hw.n_gpus;
    dc.pipeline_depth = o.depth;
    // Frames: the LIFO pools keep the highest slot id at the peak concurrent
    // use, which never exceeds every request of the trace held at once.
    const std::int64_t bound = tr.all_blocks * m.n_layers;
    dc.gpu_slots = std::min(cfg.pools.gpu_blocks_total, bound);
    const std::int64_t host_need = cfg.layerkv ? std::min(cfg.pools.cpu_blocks_total, bound) : 1;
    dc.host_slots = o.host_slots > 0 ? std::min(o.host_slots, host_need) : host_need;
    const std::int64_t batch_blocks = (std::max<std::int64_t>(cfg.max_batch_tokens, tr.max_total) + bs - 1) / bs;
    max_batch_ = std::max(1, tr.n);
    dc.arena_slots = batch_blocks + max_batch_ + 16;
    dc.max_requests = tr.n + 1;
    dc.max_blocks = static_cast<int>((tr.max_total + bs - 1) / bs + 2);
    dc.max_batch = max_batch_;
    dc.staging_chunks = 16;
    dc.chunk_bytes = static_cast<std::int64_t>(cfg.chunk_bytes);
    dc.pinned_frames = o.pinned_frames > 0 ? std::min(o.pinned_frames, dc.host_slots) : 0;
    SERVE_CUDA(cudaSetDevice(o.device));
    SERVE_LKV(lkv_device_create(&ms, bs, &dc, &dev_));
    lkv::device_bind_manager(dev_, kv_);
    lkv_device_info info{};
    SERVE_LKV(lkv_device_get_info(dev_, &info));
    cs_ = static_cast<cudaStream_t>(info.compute_stream);
    hl_ = info.kv_heads_local;
    hq_ = info.q_heads_local;
    d_ = info.head_dim;
    T_ = tr.max_prompt;
    // prefill activations and K/V, decode rows
    alloc(&q_, T_ * hq_ * d_);
    alloc(&out_, T_ * hq_ * d_);
    alloc(&k_, T_ * hl_ * d_);
    alloc(&v_, T_ * hl_ * d_);
    alloc(&dq_, static_cast<std::int64_t>(max_batch_) * hq_ * d_);
    alloc(&dout_, static_cast<std::int64_t>(max_batch_) * hq_ * d_);
    alloc(&dk_, static_cast<std::int64_t>(max_batch_) * hl_ * d_);
    alloc(&dv_, static_cast<std::int64_t>(max_batch_) * hl_ * d_);
    fill(q_, T_ * hq_ * d_, 11, 2.0f);
    fill(dq_, static_cast<std::int64_t>(max_batch_) * hq_ * d_, 12, 2.0f);
    if (o_.dense) {
      hid_ = m.hidden;
      qkv_ = m.hidden + 2ll * m.n_kv_heads * m.d_head;
      ffn_ = o.ffn;
      if (ffn_ <= 0) {  // n_param / L ~ hidden*qkv + hidden^2 + 3*hidden*ffn (embeddings ignored)
        const double per_layer = m.n_param / m.n_layers;
        const double rest = per_layer - static_cast<double>(hid_) * qkv_ - static_cast<double>(hid_) * hid_;
        ffn_ = std::max<std::int64_t>(256, static_cast<std::int64_t>(rest / (3.0 * hid_)) / 256 * 256);
      }
      const std::int64_t wmax = std::max({hid_ * qkv_, hid_ * hid_, hid_ * 2 * ffn_, ffn_ * hid_});
      alloc(&w_, wmax);
      const std::int64_t rows = std::max<std::int64_t>(T_, max_batch_);
      alloc(&x_, rows * hid_);
      alloc(&y_, rows * std::max({qkv_, 2 * ffn_, hid_}));
      fill(w_, wmax, 13, 0.04f);
      fill(x_, rows * hid_, 14, 2.0f);
      SERVE_BLAS(cublasCreate(&blas_));
      SERVE_BLAS(cublasSetStream(blas_, cs_));
    }
    SERVE_CUDA(cudaEventCreate(&base_));
    SERVE_CUDA(cudaEventCreate(&ev0_));
    SERVE_CUDA(cudaEventCreate(&ev1_));
    SERVE_CUDA(cudaEventCreate(&probe_));
    SERVE_CUDA(cudaStreamCreateWithFlags(&probe_s_, cudaStreamNonBlocking));
    SERVE_CUDA(cudaDeviceSynchronize());
    SERVE_CUDA(cudaEventRecord(base_, probe_s_));
    SERVE_CUDA(cudaEventSynchronize(base_));
  }

  ~DeviceExecutor() override {
    cudaSetDevice(o_.device);
    if (dev_) lkv_device_synchronize(dev_);
    if (blas_) cublasDestroy(blas_);
    for (void* p : bufs_) cudaFree(p);
    for (cudaEvent_t e : {base_, ev0_, ev1_, probe_})
      if (e) cudaEventDestroy(e);
    if (probe_s_) cudaStreamDestroy(probe_s_);
    if (dev_) lkv_device_destroy(dev_);  // unbinds from the manager
  }

  // ---- Executor
  double prefill(std::int64_t id, std::int64_t prompt, const std::vector<int>& offloaded, double now) override {
    const double modelled = modelled_.prefill(id, prompt, offloaded, now);
    if (prompt > T_) throw lkv::CapacityError("serve: prompt longer than the executor's buffers");
    const float scale = 1.0f / std::sqrt(static_cast<float>(d_));
    SERVE_CUDA(cudaEventRecord(ev0_, cs_));
    for (int l = 0; l < cfg_.model.n_layers; ++l) {
      // QKV projection -> the layer's K/V exist: pack + D2H them right away so
      // the copy overlaps this layer's attention and MLP
      if (o_.dense) qkv_gemm(prompt);
      SERVE_LKV(lkv_fill_kv(dev_, k_, v_, prompt, 0, l, o_.kv_seed, cs_));
      SERVE_LKV(lkv_prefill_layer(dev_, id, l, k_, v_, prompt, cs_));
      if (o_.attention) SERVE_LKV(lkv_prefill_attention(dev_, q_, k_, v_, out_, prompt, scale, LKV_DTYPE_BF16, cs_));
      if (o_.dense) rest_gemms(prompt);
      launches_ += 1 + (o_.dense ? 4 : 0) + (o_.attention ? 1 : 0) + 2;  // fill, gemms, attention, table + scatter/pack
    }
    SERVE_CUDA(cudaEventRecord(ev1_, cs_));
    const double dev_s = span_s();
    prefill_s_ += dev_s;
    ++prefills_;
    return o_.measured ? stamp(ev1_) : modelled;
  }

  double offload(const layersim::OffloadJob& job, double now) override {
    const double modelled = modelled_.offload(job, now);  // counts the job; the D2H already runs (observer)
    if (!o_.measured) return modelled;
    pending_.push_back(job.job_id);
    return std::numeric_limits<double>::quiet_NaN();
  }

  double decode(const std::vector<std::int64_t>& batch, std::int64_t batch_kv, double now) override {
    const double modelled = modelled_.decode(batch, batch_kv, now);
    const int n = static_cast<int>(batch.size());
    if (n > max_batch_) throw lkv::CapacityError("serve: decode batch larger than the executor's rows");
    pos_.resize(static_cast<std::size_t>(n));
    for (int m = 0; m < n; ++m) pos_[static_cast<std::size_t>(m)] = kv_.request(batch[static_cast<std::size_t>(m)]).cached_tokens;
    const float scale = 1.0f / std::sqrt(static_cast<float>(d_));
    SERVE_CUDA(cudaEventRecord(ev0_, cs_));
    SERVE_LKV(lkv_decode_begin_append(dev_, batch.data(), n));
    for (int l = 0; l < cfg_.model.n_layers; ++l) {
      SERVE_LKV(lkv_fill_kv_tokens(dev_, dk_, dv_, pos_.data(), n, l, o_.kv_seed, cs_));
      if (o_.dense) dense(n);
      SERVE_LKV(lkv_decode_append_layer(dev_, l, dk_, dv_, cs_));
      SERVE_LKV(lkv_decode_layer(dev_, l, dq_, dout_, scale, LKV_DTYPE_BF16, cs_));
      launches_ += 1 + (o_.dense ? 4 : 0);
    }
    SERVE_LKV(lkv_decode_end(dev_));
    lkv_decode_stats st{};
    SERVE_CUDA(cudaEventRecord(ev1_, cs_));
    const double dev_s = span_s();
    if (lkv_decode_last_stats(dev_, &st) == LKV_OK) launches_ += st.kernel_launches;
    decode_s_ += dev_s;
    ++decodes_;
    return o_.measured ? stamp(ev1_) : modelled;
  }

  void transfer_totals(std::int64_t* a, double* b, std::int64_t* c, double* d) const override {
    modelled_.transfer_totals(a, b, c, d);
  }
  // the virtual clock's schedule (the one the device executes); none when
  // CUDA events are the clock
  const std::vector<layersim::TransferLogRow>* transfer_log() const override {
    return o_.measured ? nullptr : modelled_.transfer_log();
  }

  void before_release(std::int64_t id) override {
    if (!o_.verify) return;
    std::int64_t bad = 0;
    SERVE_LKV(lkv_verify_request(dev_, id, kv_.request(id).cached_tokens, o_.kv_seed, &bad));
    mismatched_ += bad;
    ++verified_;
  }

  bool measured() const override { return o_.measured; }
  double clock() override {
    SERVE_CUDA(cudaEventRecord(probe_, probe_s_));
    return stamp(probe_);
  }
  void skip_to(double t) override {
    const double c = clock();
    if (t > c) skip_ += t - c;
  }
  bool offloads_pending() const override { return !pending_.empty(); }
  void poll_offloads(bool wait, std::vector<std::pair<double, std::int64_t>>* done) override {
    while (!pending_.empty()) {
      const std::int64_t job = pending_.front();
      cudaEvent_t ev = lkv::device_job_event(dev_, job);
      if (!ev) throw layersim::SimulationError("serve: escalation job " + std::to_string(job) + " has no copy event");
      if (wait) {
        SERVE_CUDA(cudaEventSynchronize(ev));
        wait = false;
      } else if (cudaEventQuery(ev) != cudaSuccess) {
        cudaGetLastError();
        return;
      }
      done->emplace_back(stamp(ev), job);
      pending_.pop_front();
    }
  }

  // ---- stats
  std::int64_t prefills_ = 0, decodes_ = 0, mismatched_ = 0, verified_ = 0, launches_ = 0;
  double prefill_s_ = 0, decode_s_ = 0;

 private:
  void alloc(__nv_bfloat16** p, std::int64_t elems) {
    void* q = nullptr;
    SERVE_CUDA(cudaMalloc(&q, static_cast<std::size_t>(std::max<std::int64_t>(elems, 1)) * 2));
    bufs_.push_back(q);
    *p = static_cast<__nv_bfloat16*>(q);
  }
  void fill(__nv_bfloat16* p, std::int64_t n, unsigned long long seed, float scale) {
    fill_uniform_bf16<<<592, 256, 0, cs_>>>(p, n, seed, scale);
    SERVE_CUDA(cudaGetLastError());
  }
  // Row-major Y[M, N] = X[M, K] W[K, N] as column-major Y^T = W^T X^T.
  void gemm(const __nv_bfloat16* X, const __nv_bfloat16* W, __nv_bfloat16* Y, std::int64_t M, std::int64_t N,
            std::int64_t K) {
    const float one = 1.0f, zero = 0.0f;
    SERVE_BLAS(cublasGemmEx(blas_, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(N), static_cast<int>(M),
                            static_cast<int>(K), &one, W, CUDA_R_16BF, static_cast<int>(N), X, CUDA_R_16BF,
                            static_cast<int>(K), &zero, Y, CUDA_R_16BF, static_cast<int>(N), CUBLAS_COMPUTE_32F,
                            CUBLAS_GEMM_DEFAULT));
  }
  // The layer's projections and MLP: QKV, O, gate+up, down (norms, RoPE and
  // the SiLU product are elementwise and left out).
  void qkv_gemm(std::int64_t M) { gemm(x_, w_, y_, M, qkv_, hid_); }
  void rest_gemms(std::int64_t M) {  // O projection, gate+up, down
    gemm(x_, w_, y_, M, hid_, hid_);
    gemm(x_, w_, y_, M, 2 * ffn_, hid_);
    gemm(y_, w_, x_, M, hid_, ffn_);
  }
  void dense(std::int64_t M) {
    qkv_gemm(M);
    rest_gemms(M);
  }
  double span_s() {
    SERVE_CUDA(cudaEventSynchronize(ev1_));
    float ms = 0.f;
    SERVE_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
    return ms / 1e3;
  }
  // Engine time of a completed event: device time since start + idle skips.
  double stamp(cudaEvent_t ev) {
    SERVE_CUDA(cudaEventSynchronize(ev));
    float ms = 0.f;
    SERVE_CUDA(cudaEventElapsedTime(&ms, base_, ev));
    return ms / 1e3 + skip_;
  }

  const lkv::ServeConfig& cfg_;
  layersim::KvManager& kv_;
  DeviceOptions o_;
  lkv::ModelledExecutor modelled_;
  lkv_device* dev_ = nullptr;
  cudaStream_t cs_ = nullptr, probe_s_ = nullptr;
  cublasHandle_t blas_ = nullptr;
  cudaEvent_t base_ = nullptr, ev0_ = nullptr, ev1_ = nullptr, probe_ = nullptr;
  std::vector<void*> bufs_;
  __nv_bfloat16 *q_ = nullptr, *out_ = nullptr, *k_ = nullptr, *v_ = nullptr;
  __nv_bfloat16 *dq_ = nullptr, *dout_ = nullptr, *dk_ = nullptr, *dv_ = nullptr;
  __nv_bfloat16 *w_ = nullptr, *x_ = nullptr, *y_ = nullptr;
  std::int64_t hid_ = 0, qkv_ = 0, ffn_ = 0, T_ = 0;
  int hl_ = 0, hq_ = 0, d_ = 0, max_batch_ = 1;
  std::vector<std::int64_t> pos_;
  std::deque<std::int64_t> pending_;
  double skip_ = 0.0;
};

lkv::ServeConfig to_serve_config(const lkv_serve_config* c) {
  lkv::ServeConfig e;
  e.model = lkv::to_model(&c->model);
  e.hw.flops = c->hw.flops;
  e.hw.hbm_bandwidth = c->hw.hbm_bandwidth;
  e.hw.pcie_bandwidth = c->hw.pcie_bandwidth;
  e.hw.nvlink = c->hw.nvlink != 0;
  e.hw.n_gpus = c->hw.n_gpus;
  e.hw.gpu_mem = c->hw.gpu_mem;
  e.hw.kv_reserve_fraction = c->hw.kv_reserve_fraction;
  e.cost = {c->cost.alpha, c->cost.beta, c->cost.gamma, c->cost.delta};
  e.slo = {c->ttft_slo, c->tpot_slo};
  e.layerkv = c->policy_layerkv != 0;
  e.slo_scheduler = c->slo_scheduler != 0;
  e.pools = {c->gpu_blocks, c->cpu_blocks, c->tokens_per_block};
  e.threshold_fraction = c->threshold_fraction;
  e.horizon = c->horizon;
  e.predictor_accuracy = c->predictor_accuracy;
  e.max_batch_tokens = c->max_batch_tokens;
  e.max_time = c->max_time;
  e.chunk_bytes = c->chunk_bytes;
  e.seed = c->seed;
  e.force_retained_layers = c->force_retained_layers;
  e.invariant_checks = c->invariant_checks != 0;
  return e;
}

lkv::Trace to_trace(int32_t n, const int64_t* ids, const double* arrival, const int32_t* prompt, const int32_t* output,
                    std::uint64_t seed) {
  lkv::Trace t;
  t.seed = seed;
  t.requests.resize(static_cast<std::size_t>(n));
  for (int32_t i = 0; i < n; ++i) t.requests[static_cast<std::size_t>(i)] = {ids[i], arrival[i], prompt[i], output[i]};
  return t;
}

void from_trace(const lkv::Trace& t, int64_t* ids, double* arrival, int32_t* p, int32_t* o, std::size_t cap) {
  for (std::size_t i = 0; i < t.requests.size() && i < cap; ++i) {
    ids[i] = t.requests[i].id;
    arrival[i] = t.requests[i].arrival;
    p[i] = t.requests[i].prompt_tokens;
    o[i] = t.requests[i].output_tokens;
  }
}

}  // namespace

#define SERVE_TRY try {
#define SERVE_CATCH                              \
  }                                              \
  catch (...) {                                  \
    return lkv::status_from_current_exception(); \
  }                                              \
  return LKV_OK;

int lkv_serve_run(const lkv_serve_config* c, int32_t n, const int64_t* ids, const double* arrival,
                  const int32_t* prompt, const int32_t* output, lkv_serve_summary* out, lkv_serve_request_row* rows,
                  int32_t rows_cap) {
  return lkv_serve_run_ex(c, n, ids, arrival, prompt, output, out, rows, rows_cap, nullptr, 0, nullptr, nullptr, 0,
                          nullptr);
}

int lkv_serve_run_ex(const lkv_serve_config* c, int32_t n, const int64_t* ids, const double* arrival,
                     const int32_t* prompt, const int32_t* output, lkv_serve_summary* out, lkv_serve_request_row* rows,
                     int32_t rows_cap, char* tlog, size_t tlog_cap, size_t* tlog_len, char* dlog, size_t dlog_cap,
                     size_t* dlog_len) {
  if (!c || !out || n < 1 || !ids || !arrival || !prompt || !output || (tlog && !tlog_len) || (dlog && !dlog_len)) {
    lkv::set_error("invalid argument: lkv_serve_run");
    return LKV_ERR_INVALID;
  }
  SERVE_TRY
  const lkv::ServeConfig cfg = to_serve_config(c);
  lkv::Trace trace = to_trace(n, ids, arrival, prompt, output, c->seed);
  DeviceExecutor* dexec = nullptr;
  lkv::ServeEngine::ExecutorFactory factory = nullptr;
  if (c->executor != LKV_SERVE_MODELLED) {
    DeviceOptions o;
    o.measured = c->executor == LKV_SERVE_DEVICE_MEASURED;
    o.dense = c->dense_gemms != 0;
    o.attention = c->prefill_attention != 0;
    o.verify = c->verify_kv != 0;
    o.device = c->device;
    o.depth = std::max(1, c->pipeline_depth);
    o.ffn = c->ffn;
    o.host_slots = c->host_slots;
    o.kv_seed = c->kv_seed;
    o.tp_rank = c->tp_rank;
    o.pinned_frames = c->pinned_frames;
    if (c->tp_rank < 0 || c->tp_rank >= std::max(1, c->hw.n_gpus)) {
      lkv::set_error("invalid argument: lkv_serve_run tp_rank outside [0, hw.n_gpus)");
      return LKV_ERR_INVALID;
    }
    TraceShape shape;
    shape.n = n;
    for (const auto& r : trace.requests) {
      shape.max_prompt = std::max<std::int64_t>(shape.max_prompt, r.prompt_tokens);
      const std::int64_t total = static_cast<std::int64_t>(r.prompt_tokens) + r.output_tokens;
      shape.max_total = std::max<std::int64_t>(shape.max_total, total);
      shape.all_blocks += (total + c->tokens_per_block - 1) / c->tokens_per_block + 1;
    }
    factory = [o, shape, &dexec](const lkv::ServeConfig& sc, layersim::KvManager& kv) {
      auto e = std::make_unique<DeviceExecutor>(sc, kv, o, shape);
      dexec = e.get();
      return std::unique_ptr<lkv::Executor>(std::move(e));
    };
  }
  lkv::ServeEngine engine(cfg, std::move(trace), factory);
  const lkv::ServeReport r = engine.run();
  std::memset(out, 0, sizeof *out);
  out->mean_ttft = r.mean_ttft;
  out->p50_ttft = r.p50_ttft;
  out->p99_ttft = r.p99_ttft;
  out->mean_tpot = r.mean_tpot;
  out->throughput = r.throughput_tokens_per_s;
  out->makespan = r.makespan;
  out->d2h_jobs = r.d2h_jobs;
  out->h2d_jobs = r.h2d_jobs;
  out->d2h_bytes = r.d2h_bytes;
  out->h2d_bytes = r.h2d_bytes;
  out->completed = r.completed;
  out->n_rows = static_cast<int32_t>(r.requests.size());
  out->violations = r.violations;
  out->escalations = r.escalations;
  if (dexec) {
    out->prefills = dexec->prefills_;
    out->decode_iterations = dexec->decodes_;
    out->kv_words_mismatched = dexec->mismatched_;
    out->requests_verified = dexec->verified_;
    out->gpu_kernel_launches = dexec->launches_;
    out->prefill_device_s = dexec->prefill_s_;
    out->decode_device_s = dexec->decode_s_;
  }
  if (rows) {
    for (std::size_t i = 0; i < r.requests.size() && static_cast<int32_t>(i) < rows_cap; ++i) {
      const auto& q = r.requests[i];
      rows[i] = {q.id, q.arrival, q.queuing, q.prefill, q.ttft, q.mean_tpot, q.output_tokens, q.violated ? 1 : 0};
    }
  }
  const auto put = [](const std::string& s, char* buf, size_t cap, size_t* len) {
    if (!len) return;
    *len = s.size();
    if (buf && cap > s.size()) {
      std::memcpy(buf, s.data(), s.size());
      buf[s.size()] = 0;
    }
  };
  put(r.transfer_log_csv(), tlog, tlog_cap, tlog_len);
  put(r.decision_log_csv(), dlog, dlog_cap, dlog_len);
  SERVE_CATCH
}

int lkv_serve_requests_csv(const lkv_serve_request_row* rows, int32_t n, char* buf, size_t cap, size_t* len) {
  if ((!rows && n > 0) || !len) {
    lkv::set_error("invalid argument: lkv_serve_requests_csv");
    return LKV_ERR_INVALID;
  }
  SERVE_TRY lkv::ServeReport rep;
  rep.requests.resize(static_cast<std::size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    auto& q = rep.requests[static_cast<std::size_t>(i)];
    q.id = rows[i].id;
    q.arrival = rows[i].arrival;
    q.queuing = rows[i].queuing;
    q.prefill = rows[i].prefill;
    q.ttft = rows[i].ttft;
    q.mean_tpot = rows[i].mean_tpot;
    q.output_tokens = rows[i].output_tokens;
    q.violated = rows[i].violated != 0;
  }
  const std::string s = rep.requests_csv();
  *len = s.size();
  if (buf && cap > s.size()) {
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = 0;
  }
  SERVE_CATCH
}

int lkv_trace_generate(int32_t sharegpt, int32_t n, int32_t prompt, int32_t output, double rate, uint64_t seed,
                       int64_t* ids, double* arrival, int32_t* p, int32_t* o) {
  if (!ids || !arrival || !p || !o) {
    lkv::set_error("invalid argument: lkv_trace_generate");
    return LKV_ERR_INVALID;
  }
  SERVE_TRY const lkv::Trace t =
      sharegpt ? lkv::trace_sharegpt_like(n, rate, seed) : lkv::trace_fixed(n, prompt, output, rate, seed);
  from_trace(t, ids, arrival, p, o, static_cast<std::size_t>(n));
  SERVE_CATCH
}

int lkv_trace_read_jsonl(const char* path, int64_t* ids, double* arrival, int32_t* p, int32_t* o, int32_t cap,
                         int32_t* n, int32_t* unsorted) {
  if (!path || !n) {
    lkv::set_error("invalid argument: lkv_trace_read_jsonl");
    return LKV_ERR_INVALID;
  }
  SERVE_TRY bool uns = false;
  const lkv::Trace t = lkv::read_trace_jsonl(path, &uns);
  *n = static_cast<int32_t>(t.requests.size());
  if (unsorted) *unsorted = uns;
  if (ids && arrival && p && o) from_trace(t, ids, arrival, p, o, static_cast<std::size_t>(std::max(cap, 0)));
  SERVE_CATCH
}

int lkv_trace_write_jsonl(const char* path, int32_t n, const int64_t* ids, const double* arrival, const int32_t* p,
                          const int32_t* o) {
  if (!path || n < 0 || (n > 0 && (!ids || !arrival || !p || !o))) {
    lkv::set_error("invalid argument: lkv_trace_write_jsonl");
    return LKV_ERR_INVALID;
  }
  SERVE_TRY lkv::write_trace_jsonl(to_trace(n, ids, arrival, p, o, 0), path);
  SERVE_CATCH
}
