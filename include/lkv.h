/*
 * lkv.h — C ABI of the B200-native LayerKV data-movement path.
 *
 * The reference (arXiv 2410.00428 artifact, "layersim") has no C ABI: its
 * boundary is the C++ API of the static library layersim_core. This header is
 * the thin, FFI-bindable layer under the C++ drop-in (include/layersim/ headers):
 * plain structs, pointers and sizes, no C++ or torch types. Every entry point
 * names the reference interface it replaces (paths relative to
 * /root/reference/proj). INTEGRATION.md shows the ctypes binding a
 * maintainer would add and where engine.cpp calls into the device half.
 *
 * Error convention (reference errors.hpp:9-17 + kv_manager.hpp:94-150):
 *   capacity failures are VALUES (ok flags / has_value = 0), exactly where the
 *   reference returns false / std::nullopt; logic errors are negative status
 *   codes where the reference throws, with the exception text available from
 *   lkv_last_error() (thread-local).
 */
#ifndef LKV_H_
#define LKV_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define LKV_API __attribute__((visibility("default")))
#else
#define LKV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define LKV_OK 0
#define LKV_ERR_SIMULATION (-1) /* layersim::SimulationError */
#define LKV_ERR_CONFIG (-2)     /* layersim::ConfigError */
#define LKV_ERR_DOMAIN (-3)     /* std::domain_error */
#define LKV_ERR_INVALID (-4)    /* std::invalid_argument / bad C argument */
#define LKV_ERR_CUDA (-5)       /* CUDA runtime failure on the device path */
#define LKV_ERR_CAPACITY (-6)   /* a device/host arena is too small */
#define LKV_ERR_INTERNAL (-7)

LKV_API const char* lkv_last_error(void);
/* Build identification: "lkv <version> sm_100a" (also proves the .so loaded). */
LKV_API const char* lkv_version(void);

/* ---- value types (reference cost_model.hpp:9-43, kv_manager.hpp:13-78) --- */
typedef struct lkv_model_spec {
  int32_t n_layers, n_heads, n_kv_heads, d_head;
  int64_t hidden;
  double n_param;
  int32_t f_precision;
  int32_t pad_;
} lkv_model_spec;

typedef struct lkv_hardware_spec {
  double flops, hbm_bandwidth, pcie_bandwidth;
  int32_t nvlink, n_gpus;
  double gpu_mem, kv_reserve_fraction;
} lkv_hardware_spec;

typedef struct lkv_cost_params {
  double alpha, beta, gamma, delta;
} lkv_cost_params;

typedef struct lkv_pool_sizing {
  int64_t max_input_tokens;
  int32_t tokens_per_block;
  int32_t pad_;
  double activation_layers_factor, cpu_pool_multiple;
} lkv_pool_sizing;

typedef struct lkv_block_pools {
  int64_t gpu_blocks_total, cpu_blocks_total;
  int32_t tokens_per_block;
  int32_t pad_;
} lkv_block_pools;

typedef struct lkv_offload_job {
  int64_t job_id, request_id;
  double bytes;
  int32_t layer_count;
  int32_t pad_;
  int64_t gpu_blocks;
} lkv_offload_job;

typedef struct lkv_fetch_job {
  int32_t layer;
  int32_t pad_;
  double bytes;
} lkv_fetch_job;

typedef struct lkv_freed_counts {
  int64_t gpu, cpu, deferred_gpu;
} lkv_freed_counts;

#define LKV_LOC_NONE 0
#define LKV_LOC_GPU 1
#define LKV_LOC_CPU 2
typedef struct lkv_slot_loc { /* reference kv_manager.hpp:44-49 */
  uint8_t loc;
  uint8_t offload_in_flight;
  uint16_t pad_;
  uint32_t slot;
  uint32_t dest_slot;
} lkv_slot_loc;

#define LKV_OFFLOAD_HALF 0
#define LKV_OFFLOAD_FULL 1

/* ---- cost model (reference cost_model.hpp:48-78) ------------------------ */
LKV_API int lkv_model_validate(const lkv_model_spec* m);
LKV_API int lkv_kv_bytes_per_token_layer(const lkv_model_spec* m, int64_t* out);
LKV_API int lkv_prefill_time(const lkv_model_spec*, const lkv_hardware_spec*, const lkv_cost_params*,
                     int64_t seqlen, double* out);
LKV_API int lkv_offload_time(const lkv_model_spec*, const lkv_hardware_spec*, const lkv_cost_params*,
                     int64_t seqlen, int32_t layers_offloaded, double* out);
LKV_API int lkv_min_retained_layers(const lkv_model_spec*, const lkv_hardware_spec*,
                            const lkv_cost_params*, int64_t seqlen, int32_t* out);
LKV_API int lkv_decode_step_time(const lkv_model_spec*, const lkv_hardware_spec*, const lkv_cost_params*,
                         int64_t batch_kv_tokens, double* out);
LKV_API int lkv_allreduce_time(const lkv_model_spec*, const lkv_hardware_spec*, int64_t tokens,
                       double* out);

/* ---- pool sizing / placement (reference kv_manager.hpp:27-40) ---------- */
LKV_API int lkv_pool_size_from_hardware(const lkv_model_spec*, const lkv_hardware_spec*,
                                const lkv_pool_sizing*, lkv_block_pools* out);
/* retained[x], offloaded[n_layers - x] */
LKV_API int lkv_layer_placement(int32_t n_layers, int32_t x, int32_t* retained, int32_t* offloaded);

/* ---- KvManager (reference kv_manager.hpp:80-150) ------------------------ */
typedef struct lkv_kv_manager lkv_kv_manager;

typedef struct lkv_kv_stats {
  int64_t gpu_blocks_total, gpu_blocks_free, cpu_blocks_total, cpu_blocks_free;
  int32_t tokens_per_block, n_layers;
  int64_t pending_offloads, live_requests;
} lkv_kv_stats;

LKV_API int lkv_kv_create(const lkv_block_pools* pools, const lkv_model_spec* model, lkv_kv_manager** out);
LKV_API int lkv_kv_destroy(lkv_kv_manager* kv);
LKV_API int lkv_kv_stats_get(const lkv_kv_manager* kv, lkv_kv_stats* out);
LKV_API int lkv_kv_blocks_per_layer(const lkv_kv_manager*, int64_t tokens, int64_t* out);
LKV_API int lkv_kv_request_wise_gpu_blocks(const lkv_kv_manager*, int64_t prompt_tokens, int64_t* out);
LKV_API int lkv_kv_allocate_prefill(lkv_kv_manager*, int64_t request_id, int64_t prompt_tokens, int32_t x,
                            int32_t* ok);
LKV_API int lkv_kv_has_request(const lkv_kv_manager*, int64_t request_id, int32_t* out);
/* request(id): sizes first, then the table (entries block-major: [b * L + l]). */
LKV_API int lkv_kv_request_shape(const lkv_kv_manager*, int64_t request_id, int64_t* cached_tokens,
                         int64_t* n_blocks);
LKV_API int lkv_kv_request_table(const lkv_kv_manager*, int64_t request_id, lkv_slot_loc* entries,
                         int64_t* token_begin, uint8_t* layer_residency);
LKV_API int lkv_kv_retained_layer_count(const lkv_kv_manager*, int64_t request_id, int32_t* out);
LKV_API int lkv_kv_gpu_blocks_held(const lkv_kv_manager*, int64_t request_id, int64_t* out);
LKV_API int lkv_kv_gpu_row_cost(const lkv_kv_manager*, int64_t request_id, int64_t* out);
LKV_API int lkv_kv_cpu_row_cost(const lkv_kv_manager*, int64_t request_id, int64_t* out);
LKV_API int lkv_kv_offload_reclaim(const lkv_kv_manager*, int64_t request_id, int32_t mode, int64_t* out);
LKV_API int lkv_kv_plan_offload(lkv_kv_manager*, int64_t request_id, int32_t mode, lkv_offload_job* job,
                        int32_t* has_value);
LKV_API int lkv_kv_complete_offload(lkv_kv_manager*, int64_t job_id);
/* Writes min(cap, count) jobs; *count = number of jobs (call with cap 0 to size). */
LKV_API int lkv_kv_plan_decode_fetch(const lkv_kv_manager*, int64_t request_id, lkv_fetch_job* out,
                             int32_t cap, int32_t* count);
LKV_API int lkv_kv_needs_append(const lkv_kv_manager*, int64_t request_id, int32_t* out);
LKV_API int lkv_kv_append_decode_block(lkv_kv_manager*, int64_t request_id, int32_t* ok);
LKV_API int lkv_kv_note_token(lkv_kv_manager*, int64_t request_id);
LKV_API int lkv_kv_release(lkv_kv_manager*, int64_t request_id, lkv_freed_counts* out);
LKV_API int lkv_kv_check_conservation(const lkv_kv_manager*);
/* dump_table text. *len = bytes needed (no NUL); written when cap > *len. */
LKV_API int lkv_kv_dump_table(const lkv_kv_manager*, char* buf, size_t cap, size_t* len);
/* FNV-1a-64 of the dump_table text (the parity hash of BASELINE.md §2). */
LKV_API int lkv_kv_dump_hash(const lkv_kv_manager*, uint64_t* out);
/* One LIFO free list (which: 0 = GPU, 1 = CPU) as the reference's SlotPool
 * keeps it (free_stack_, kv_manager.hpp:153-166, kv_manager.cpp:52-74): the
 * whole stack bottom to top (next alloc = last). *size = free slots; the stack
 * is written to out when cap >= *size. */
LKV_API int lkv_kv_free_stack(const lkv_kv_manager*, int32_t which, uint32_t* out, int64_t cap, int64_t* size);
/* The free-list journal the device mirror consumes (lkv_device_bind owns it
 * while a device is bound; call it only on an unbound manager): the change
 * since the previous take as {next_fresh, low, size, changed} plus the
 * pushed entries [low, size), written to out when cap >= size - low. A
 * mirror applies it as: stack = [total-1 ... next_fresh] + pushed[0..size),
 * with pushed[low..size) replaced. full = 1 restarts from low = 0. */
LKV_API int lkv_kv_free_delta(lkv_kv_manager*, int32_t which, int32_t full, int64_t* next_fresh, int64_t* low,
                              int64_t* size, int32_t* changed, uint32_t* out, int64_t cap);

/* ---- PcieBus, parity-mode timing (reference interconnect.hpp:9-80) ------ */
typedef struct lkv_pcie_bus lkv_pcie_bus;
#define LKV_D2H 0
#define LKV_H2D 1
typedef struct lkv_transfer_schedule {
  double start, completion;
  int32_t chunks, deferrals;
} lkv_transfer_schedule;
typedef struct lkv_span {
  double begin, end;
  int32_t is_allreduce;
  int32_t pad_;
} lkv_span;

LKV_API int lkv_bus_create(double delta, lkv_pcie_bus** out);
LKV_API int lkv_bus_destroy(lkv_pcie_bus*);
LKV_API int lkv_bus_register_allreduce(lkv_pcie_bus*, double start, double duration,
                               const lkv_hardware_spec* hw);
LKV_API int lkv_bus_submit_transfer(lkv_pcie_bus*, double bytes, int32_t direction, double submit_time,
                            double chunk_bytes, const lkv_hardware_spec* hw,
                            lkv_transfer_schedule* out);
LKV_API int lkv_bus_state(const lkv_pcie_bus*, double t, double* busy_until, double* allreduce_busy_until,
                  int32_t* allreduce_active_at_t);
LKV_API int lkv_bus_enable_history(lkv_pcie_bus*, int32_t on);
LKV_API int lkv_bus_chunk_history(const lkv_pcie_bus*, lkv_span* out, int32_t cap, int32_t* count);
LKV_API int lkv_bus_allreduce_windows(const lkv_pcie_bus*, lkv_span* out, int32_t cap, int32_t* count);

/* schedule_prefill_span (reference engine.hpp:59-71, engine.cpp:22-45). */
LKV_API int lkv_schedule_prefill_span(const lkv_model_spec*, const lkv_hardware_spec*,
                              const lkv_cost_params*, lkv_pcie_bus*, const int32_t* offloaded,
                              int32_t n_offloaded, int64_t prompt_tokens, double start,
                              double chunk_bytes, int32_t transfers_enabled, double* completion,
                              lkv_transfer_schedule* jobs, int32_t cap, int32_t* n_jobs);

/* ======================================================================== *
 * Device half (sm_100a). Replaces what the reference only models:
 *   per-layer prefill KV write + D2H job   engine.cpp:35-42 (schedule_prefill_span)
 *   escalation gather + D2H                kv_manager.cpp:222-288, engine.cpp:343-352
 *   decode H2D fetch per layer             kv_manager.cpp:290-304, engine.cpp:426-449
 *   paged decode attention                 cost_model.cpp:73-79 (decode_step_time)
 * ======================================================================== */
typedef struct lkv_device lkv_device;

typedef struct lkv_device_config {
  int32_t device;         /* CUDA ordinal */
  int32_t tp_rank;        /* KV-head shard r of tp_size: kv heads [r*Hkv/N, (r+1)*Hkv/N) */
  int32_t tp_size;
  int32_t pipeline_depth; /* decode layers whose prefetch may be in flight (>= 1) */
  int64_t gpu_slots;      /* device pool frames; must exceed the highest GPU slot id used */
  int64_t host_slots;     /* pinned host frames; must exceed the highest CPU slot id used */
  int64_t arena_slots;    /* prefetch arena frames per pipeline stage */
  int32_t max_requests;   /* device block-table rows */
  int32_t max_blocks;     /* logical blocks per request row */
  int32_t max_batch;      /* decode batch members */
  int32_t staging_chunks; /* D2H staging ring segments */
  int64_t chunk_bytes;    /* D2H staging segment size (reference TransferJob.chunk_bytes) */
  /* Tiered host memory. 0: host_slots
   * pinned frames, frame = CPU slot. > 0: every CPU slot's home is pageable
   * (host_slots of them, one MAP_NORESERVE mapping) and this many pinned,
   * device-mapped frames carry the DMA and in-kernel accesses; a cleaner
   * thread writes dirty frames home, missing slots are read in on demand. */
  int64_t pinned_frames;
} lkv_device_config;

typedef struct lkv_device_info {
  int64_t slot_bytes;   /* bytes of one (block, layer) slot on this GPU: bs * kvB / TP */
  int32_t kv_heads_local, q_heads_local, head_dim, tokens_per_block;
  void* pool;           /* device pool base, slot s at pool + s * slot_bytes */
  void* host_pool;      /* pinned host pool base, CPU slot c at host_pool + c * slot_bytes */
  void* arena;          /* device prefetch arena base */
  void* compute_stream; /* cudaStream_t: scatter, gather, table sync, attention */
  void* d2h_stream;     /* cudaStream_t: offload copies */
  void* h2d_stream;     /* cudaStream_t: prefetch copies */
  int32_t numa_node;    /* NUMA node the pinned host pool was bound to (the GPU's, sysfs); -1 none */
  int32_t gather_peers; /* gather peers on other GPUs reached over P2P (NVLink) after gather_connect */
} lkv_device_info;

/* NUMA node of CUDA device `cuda_device` (its PCI function's numa_node in
 * sysfs; -1 when unknown or single-node). Callers pin their own host buffers
 * there (the device does it for its pools). */
LKV_API int lkv_device_numa_node(int32_t cuda_device, int32_t* node);
LKV_API int lkv_device_create(const lkv_model_spec* model, int32_t tokens_per_block,
                      const lkv_device_config* cfg, lkv_device** out);
LKV_API int lkv_device_destroy(lkv_device* dev);
LKV_API int lkv_device_get_info(const lkv_device* dev, lkv_device_info* out);
/* Attach as the table observer: every KvManager mutation is mirrored into the
 * device block table and escalation jobs start their gather + D2H at
 * plan_offload (engine.cpp:345-350); complete_offload waits for the job's
 * copy to drain before the GPU send buffers are reused (engine.cpp:98-100). */
LKV_API int lkv_device_bind(lkv_device* dev, lkv_kv_manager* kv);
LKV_API int lkv_device_synchronize(lkv_device* dev);

/* Prefill layer `layer` of a request produced K and V, each
 * [tokens][kv_heads_local][head_dim] bf16 on the device (row pitch
 * kv_heads_local*head_dim elements). Retained layers are scattered into
 * their GPU slots; offloaded layers are packed into staging and streamed to
 * the pinned host frames of their CPU slots on the D2H stream — the
 * per-layer D2H job of schedule_prefill_span (engine.cpp:35-42). The
 * kernels are ordered after work already on `stream` (NULL = compute
 * stream) via an event, and later work on `stream` waits until k/v have
 * been read, so the caller may reuse them. */
LKV_API int lkv_prefill_layer(lkv_device* dev, int64_t request_id, int32_t layer, const void* k,
                      const void* v, int64_t tokens, void* stream);
/* Causal GQA prefill attention of one layer on the tcgen05 tensor cores —
 * the per-layer compute that schedule_prefill_span charges as prefill_time/L
 * (engine.cpp:27-28, cost_model.cpp:39-44) and that a layer's offload D2H
 * hides behind. q [tokens][q_heads_local][head_dim], k/v
 * [tokens][kv_heads_local][head_dim], out [tokens][q_heads_local][head_dim],
 * bf16 on the device, out in out_dtype (LKV_DTYPE_BF16 for serving,
 * LKV_DTYPE_F32 for parity checks); query row i attends keys 0..i. Runs on
 * `stream` (NULL = compute stream).
 * Input range: P.V runs in fp16 on an fp16 copy of v. Every bf16 v with
 * 2^-14 <= |v| <= 65504 converts exactly; smaller values round to fp16
 * subnormals (absolute error <= 2^-25 per value, so <= 2^-25 on the output);
 * |v| > 65504 saturates to +-65504 (no inf/NaN). q and k have no limit. */
LKV_API int lkv_prefill_attention(lkv_device* dev, const void* q, const void* k, const void* v, void* out,
                                  int64_t tokens, float scale, int32_t out_dtype, void* stream);
/* 1 when the D2H copies of an escalation job have drained. */
LKV_API int lkv_device_job_done(lkv_device* dev, int64_t job_id, int32_t* done);
/* 1 when every prefill-layer D2H issued so far for this request has drained. */
LKV_API int lkv_device_prefill_offload_done(lkv_device* dev, int64_t request_id, int32_t* done);

/* Decode iteration (engine.cpp:405-453): snapshot the batch, plan per-layer
 * fetches (plan_decode_fetch, kv_manager.cpp:290-304) and start the H2D of the
 * first pipeline_depth layers into the arena. */
LKV_API int lkv_decode_begin(lkv_device* dev, const int64_t* request_ids, int32_t n);
/* Paged attention of one layer for the batch: q is device
 * [n][q_heads_local][head_dim] bf16, out the same shape in out_dtype (bf16
 * for serving, fp32 for parity checks); kv_len of member m = its
 * cached_tokens at decode_begin. Waits for the layer's fetch, runs on the
 * compute stream, then issues the fetch of layer + pipeline_depth. `scale` =
 * softmax scale. `stream` (may be NULL) is the caller's stream: q is read
 * after the work already queued on it, and its later work sees `out`. */
#define LKV_DTYPE_BF16 0
#define LKV_DTYPE_F32 1
/* Stream arguments of the device half: NULL = the device's compute stream
 * (no ordering with any caller stream); pass cudaStreamLegacy ((void*)1) to
 * order with CUDA's legacy default stream (e.g. torch's default stream). */
LKV_API int lkv_decode_layer(lkv_device* dev, int32_t layer, const void* q, void* out, float scale,
                             int32_t out_dtype, void* stream);
LKV_API int lkv_decode_end(lkv_device* dev);

/* ---- fused all-gather of per-head decode outputs ----------
 * The path's one exchange: after each layer's decode attention every rank
 * needs every rank's per-head rows (the reference models it as the per-layer
 * all-reduce window of cost_model.cpp:81-88 / interconnect.cpp:57-61, zero on
 * NVLink). Instead of a separate collective, the split-merge kernel of
 * lkv_decode_layer stores each finished row straight into every rank's
 * gather buffer over NVLink (peer pointers) and its last CTA raises this
 * rank's epoch flag in every buffer. Rows of layer l land at
 *   gathered[l] = [max_batch][q_heads_local * tp_size][head_dim] bf16
 * (rank r's heads at column block r), double-buffered by layer parity: the
 * caller must consume gathered(l) (after lkv_decode_gather_wait) before its
 * next-but-one lkv_decode_layer.
 * Setup (once, before the first decode): each rank exports a handle, the
 * handles are exchanged out of band (e.g. torch.distributed all_gather), and
 * each rank connects with all tp_size handles in rank order. */
#define LKV_IPC_HANDLE_BYTES 64
LKV_API int lkv_device_gather_ipc_handle(lkv_device* dev, void* handle /* LKV_IPC_HANDLE_BYTES */);
LKV_API int lkv_device_gather_connect_ipc(lkv_device* dev, const void* handles /* tp_size * 64 B */,
                                          int32_t tp_size);
/* Same-process ranks (several devices in one process, or tests that put
 * every rank on one GPU): connect with the raw device pointers of each
 * rank's lkv_device_gather_buffer. */
LKV_API int lkv_device_gather_buffer(lkv_device* dev, void** base, uint64_t* bytes);
LKV_API int lkv_device_gather_connect(lkv_device* dev, void* const* bases, int32_t tp_size);
/* Enqueue on `stream` (NULL = compute stream) a wait until every rank has
 * published `layer`'s rows of the current iteration; afterwards *rows of
 * lkv_decode_gathered is readable on that stream. A rank missing for 20 s
 * traps the kernel (the context fails loudly instead of hanging). */
LKV_API int lkv_decode_gather_wait(lkv_device* dev, int32_t layer, void* stream);
LKV_API int lkv_decode_gathered(lkv_device* dev, int32_t layer, void** rows);

/* Serving decode with KV write-back. Like lkv_decode_begin,
 * but the iteration also appends each member's new token at position
 * cached_tokens (the block append_decode_block provided, engine.cpp:408-409)
 * and attention covers cached_tokens + 1 keys. The fetch booked is still
 * plan_decode_fetch's (cached tokens only). Per layer call
 * lkv_decode_append_layer before lkv_decode_layer; note_token afterwards as
 * in the reference (engine.cpp:151). */
LKV_API int lkv_decode_begin_append(lkv_device* dev, const int64_t* request_ids, int32_t n);
/* k_new/v_new [n][kv_heads_local][head_dim] bf16 on the device, members in
 * decode_begin order. The token row goes wherever its slot lives: the GPU
 * slot, or the pinned host frame of a CPU slot plus its prefetched arena copy
 * (read by this step's attention); an entry whose offload is in flight gets
 * its GPU slot and its destination frame, ordered after the in-flight D2H.
 * The reference allocates these slots (kv_manager.cpp:313-344) but never
 * schedules the bytes. `stream` orders the inputs as in lkv_decode_layer. */
LKV_API int lkv_decode_append_layer(lkv_device* dev, int32_t layer, const void* k_new, const void* v_new,
                                    void* stream);

typedef struct lkv_decode_stats {
  int64_t h2d_bytes_physical;    /* whole slots copied */
  int64_t h2d_bytes_algorithmic; /* token-exact, = sum of plan_decode_fetch bytes */
  int64_t h2d_copies;            /* cudaMemcpy(2D)Async calls */
  int64_t kv_bytes_read;         /* token-exact K+V bytes the attention consumed */
  int64_t attn_launches;
  int64_t kernel_launches;       /* every kernel this iteration launched (snapshot, attention, merge) */
  double attn_ms;                /* summed CUDA-event time of the attention launches: the attention kernel
                                    plus its PDL-overlapped split merge (one event interval per layer) */
  double h2d_ms;                 /* copy-engine busy time: summed CUDA-event time of each layer's prefetch copies */
  double iteration_ms;           /* decode_begin -> decode_end on the device */
  double h2d_span_ms;            /* first prefetch copy start -> last prefetch copy end */
  double merge_ms;               /* always 0: the merge is timed inside attn_ms (kept for ABI stability) */
  double kernel_ms;              /* attention kernels alone: first CTA start -> last warp end on %globaltimer,
                                    summed over layers (no launch latency, no merge) */
} lkv_decode_stats;
LKV_API int lkv_device_set_timing(lkv_device* dev, int32_t on);
LKV_API int lkv_decode_last_stats(const lkv_device* dev, lkv_decode_stats* out);

typedef struct lkv_offload_stats {
  int64_t d2h_bytes_physical, d2h_bytes_algorithmic, d2h_copies, jobs;
  int64_t scatter_bytes;  /* slot bytes written by the scatter kernel */
  double d2h_ms;                 /* copy-engine busy time of the D2H copies (timing on) */
  double pack_ms, scatter_ms;
} lkv_offload_stats;
LKV_API int lkv_offload_last_stats(const lkv_device* dev, lkv_offload_stats* out, int32_t reset);

/* ---- synthetic KV and verification (tests, bench, smoke) ---------------- */
/* K/V value of (layer, token, global kv head, dim): bf16 of a splitmix64
 * draw in [-1, 1), see oracle/kvgen.c for the CPU restatement. Writes
 * [tokens][kv_heads_local][head_dim] K and V for tokens [token0, token0+tokens). */
LKV_API int lkv_fill_kv(lkv_device* dev, void* k, void* v, int64_t tokens, int64_t token0, int32_t layer,
                uint64_t seed, void* stream);
/* Generator K/V of one token per row: row m (of n) is token positions[m]
 * (host array) of layer `layer`, [n][kv_heads_local][head_dim] bf16 — the
 * new tokens of a decode step in tests and the serving loop. */
LKV_API int lkv_fill_kv_tokens(lkv_device* dev, void* k, void* v, const int64_t* positions, int32_t n,
                               int32_t layer, uint64_t seed, void* stream);
/* Counts 4-byte words of the request's KV (every layer, tokens < n_tokens) that
 * differ from the generator, wherever they live now: GPU slots, or pinned
 * host frames read directly by the kernel. */
LKV_API int lkv_verify_request(lkv_device* dev, int64_t request_id, int64_t n_tokens, uint64_t seed,
                       int64_t* mismatches);
/* One CPU slot's bytes (slot_bytes) into dst, wherever they live (pinned
 * frame or pageable home); waits for in-flight copies into it. */
LKV_API int lkv_device_read_host_slot(lkv_device* dev, int64_t cpu_slot, void* dst);
/* The device mirror of one free list, read back from HBM after pending
 * journal updates are applied, in lkv_kv_free_stack's form. */
LKV_API int lkv_device_free_stack(lkv_device* dev, int32_t which, uint32_t* out, int64_t cap, int64_t* size);
typedef struct lkv_host_tier_stats {
  int64_t pinned_frames, read_in_frames, write_back_frames, evictions, hits, misses;
  int64_t staged;           /* slots whose read-in was started ahead of their prefetch */
  int64_t pin_waits;        /* prefetches that waited for a read-in still running */
  int32_t read_ahead;       /* layers staged beyond the one being fetched (last decode iteration) */
  int32_t copy_threads;     /* read-in / write-back workers */
  int64_t resident_frames;  /* frames kept resident outside the LRU order (cyclic re-fetch policy) */
} lkv_host_tier_stats;
LKV_API int lkv_device_host_tier_stats(const lkv_device* dev, lkv_host_tier_stats* out);
/* Writes generator data for every entry of a request (GPU slots and host
 * frames) without going through prefill — bench setup only. */
LKV_API int lkv_fill_request(lkv_device* dev, int64_t request_id, int64_t n_tokens, uint64_t seed);

/* ======================================================================== *
 * Serving loop and trace / CSV formats (f4).
 * The reference's caller of the path — engine.cpp's event loop with the
 * SLO-aware scheduler (scheduler.cpp), its traces (workload.cpp) and
 * requests.csv (metrics.cpp:91-101) — restated over this library. The
 * executor decides where time comes from:
 *   MODELLED         cost model + serial PcieBus: byte-identical requests.csv
 *                    to the reference (no GPU needed);
 *   DEVICE_VIRTUAL   the GPU executes every prefill / escalation / decode
 *                    iteration through the data path, the clock stays
 *                    modelled (so the schedule, and requests.csv, are the
 *                    reference's) — parity mode with real bytes;
 *   DEVICE_MEASURED  the GPU executes and CUDA events give the times:
 *                    measured TTFT / TPOT under the same scheduler.
 * ======================================================================== */
#define LKV_SERVE_MODELLED 0
#define LKV_SERVE_DEVICE_VIRTUAL 1
#define LKV_SERVE_DEVICE_MEASURED 2

typedef struct lkv_serve_config { /* reference EngineConfig, engine.hpp:32-50 */
  lkv_model_spec model;
  lkv_hardware_spec hw;
  lkv_cost_params cost;
  double ttft_slo, tpot_slo;
  int32_t policy_layerkv, slo_scheduler;
  int64_t gpu_blocks, cpu_blocks;
  int32_t tokens_per_block, horizon;
  double threshold_fraction, predictor_accuracy;
  int64_t max_batch_tokens;
  double max_time, chunk_bytes;
  uint64_t seed;
  int32_t force_retained_layers, invariant_checks;
  /* device executor */
  int32_t executor;          /* LKV_SERVE_* */
  int32_t device;            /* CUDA ordinal */
  int32_t dense_gemms;       /* per-layer QKV/O/MLP GEMMs (cuBLAS) in prefill and decode */
  int32_t prefill_attention; /* tcgen05 causal attention per prefill layer */
  int32_t verify_kv;         /* check each request's KV bit-exact vs the generator before release */
  int32_t pipeline_depth;    /* decode prefetch depth (layers) */
  int64_t ffn;               /* MLP width of the dense GEMMs; 0 = derived from n_param */
  int64_t host_slots;        /* pinned host frames; 0 = cpu_blocks */
  uint64_t kv_seed;          /* generator seed of the synthetic K/V */
  int32_t tp_rank;           /* KV-head shard the device executes (tp_size = hw.n_gpus) */
  int32_t pad_;
  int64_t pinned_frames;     /* 0: every CPU slot pinned; > 0: pageable homes + this many pinned
                                frames (the f3 tier, lkv_device_config.pinned_frames) */
} lkv_serve_config;

typedef struct lkv_serve_summary { /* MetricsReport (metrics.hpp) + transfer totals + device stats */
  double mean_ttft, p50_ttft, p99_ttft, mean_tpot, throughput, makespan;
  int64_t d2h_jobs, h2d_jobs;
  double d2h_bytes, h2d_bytes;
  int32_t completed, n_rows;
  int32_t violations, pad_;
  int64_t prefills, decode_iterations, kv_words_mismatched, requests_verified, gpu_kernel_launches;
  double prefill_device_s, decode_device_s;
  int64_t escalations; /* offload jobs planned by the escalation path */
} lkv_serve_summary;

typedef struct lkv_serve_request_row { /* one requests.csv row (metrics.hpp RequestMetrics) */
  int64_t id;
  double arrival, queuing, prefill, ttft, mean_tpot;
  int32_t output_tokens, violated;
} lkv_serve_request_row;

/* Runs the trace (arrays of n requests, ascending arrival) to completion.
 * rows (may be NULL) receives min(rows_cap, n_rows) rows in id order. */
LKV_API int lkv_serve_run(const lkv_serve_config* cfg, int32_t n, const int64_t* ids, const double* arrival,
                          const int32_t* prompt, const int32_t* output, lkv_serve_summary* out,
                          lkv_serve_request_row* rows, int32_t rows_cap);
/* lkv_serve_run plus the run's two CLI logs (tools/layersim_main.cpp:96-117):
 * transfer_log.csv over Engine::transfer_log() (engine.hpp:79,
 * interconnect.hpp:26-33) — one row per bus transfer of the virtual clock, in
 * submission order, header only under LKV_SERVE_DEVICE_MEASURED — and
 * decision_log.csv over Engine::decision_log() (engine.hpp:52-57,
 * engine.cpp:388-390) — one row per LayerKV admission round that admitted or
 * escalated. *len = bytes (no NUL), written when cap > *len; a buffer may be
 * NULL to size, a len NULL to skip that log. */
LKV_API int lkv_serve_run_ex(const lkv_serve_config* cfg, int32_t n, const int64_t* ids, const double* arrival,
                             const int32_t* prompt, const int32_t* output, lkv_serve_summary* out,
                             lkv_serve_request_row* rows, int32_t rows_cap, char* tlog, size_t tlog_cap,
                             size_t* tlog_len, char* dlog, size_t dlog_cap, size_t* dlog_len);
/* requests.csv text of rows (metrics.cpp:91-101): *len = bytes (no NUL),
 * written when cap > *len. */
LKV_API int lkv_serve_requests_csv(const lkv_serve_request_row* rows, int32_t n, char* buf, size_t cap,
                                   size_t* len);
/* generate_fixed / generate_sharegpt_like (workload.cpp:35-82), n requests. */
LKV_API int lkv_trace_generate(int32_t sharegpt, int32_t n, int32_t prompt, int32_t output, double rate,
                               uint64_t seed, int64_t* ids, double* arrival, int32_t* prompt_out,
                               int32_t* output_out);
/* load_trace (workload.cpp:84-136): *n = records; arrays (may be NULL to
 * size) receive min(cap, *n); *unsorted = 1 when input was re-sorted. */
LKV_API int lkv_trace_read_jsonl(const char* path, int64_t* ids, double* arrival, int32_t* prompt,
                                 int32_t* output, int32_t cap, int32_t* n, int32_t* unsorted);
/* save_trace (workload.cpp:138-148). */
LKV_API int lkv_trace_write_jsonl(const char* path, int32_t n, const int64_t* ids, const double* arrival,
                                  const int32_t* prompt, const int32_t* output);

#ifdef __cplusplus
}
#endif
#endif /* LKV_H_ */
