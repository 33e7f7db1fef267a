// Cost model of the LayerKV path, drop-in for the reference's
// proj/include/layersim/cost_model.hpp:9-78. Struct layouts and function
// signatures are source compatible; the formulas are evaluated in the same
// floating-point operation order so that simulated times are bit-identical.
#pragma once

#include <cstdint>

namespace layersim {

struct ModelSpec {
  int n_layers = 0;
  int n_heads = 0;
  int n_kv_heads = 0;
  int d_head = 0;
  std::int64_t hidden = 0;
  double n_param = 0.0;
  int f_precision = 0;  // bytes per KV element

  void validate() const;
};

struct HardwareSpec {
  double flops = 0.0;
  double hbm_bandwidth = 0.0;
  double pcie_bandwidth = 0.0;
  bool nvlink = false;
  int n_gpus = 1;
  double gpu_mem = 0.0;
  double kv_reserve_fraction = 0.9;

  void validate() const;
};

struct CostParams {
  double alpha = 1.0;  // prefill scale
  double beta = 1.0;   // offload scale
  double gamma = 1.0;  // decode scale
  double delta = 0.5;  // bus recheck fraction

  void validate() const;
};

// Eq. 3 (reference cost_model.cpp:39-44).
double prefill_time(const ModelSpec& model, const HardwareSpec& hw, const CostParams& p,
                    std::int64_t seqlen);
// 2 * d_head * n_kv_heads * f (reference cost_model.cpp:46-48).
std::int64_t kv_bytes_per_token_layer(const ModelSpec& model);
// Eq. 4 (reference cost_model.cpp:50-59).
double offload_time(const ModelSpec& model, const HardwareSpec& hw, const CostParams& p,
                    std::int64_t seqlen, int layers_offloaded);
// Smallest x with offload_time(L - x) <= prefill_time (reference cost_model.cpp:61-71).
int min_retained_layers(const ModelSpec& model, const HardwareSpec& hw, const CostParams& p,
                        std::int64_t seqlen);
// Memory-bound decode iteration (reference cost_model.cpp:73-79).
double decode_step_time(const ModelSpec& model, const HardwareSpec& hw, const CostParams& p,
                        std::int64_t batch_kv_tokens);
// PCIe all-reduce occupancy per layer (reference cost_model.cpp:81-88).
double allreduce_time(const ModelSpec& model, const HardwareSpec& hw, std::int64_t tokens);

}  // namespace layersim
