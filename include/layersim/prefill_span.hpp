// Per-layer prefill offload schedule, drop-in for the declaration in the
// reference's proj/include/layersim/engine.hpp:59-71 (definition
// engine.cpp:22-45). Parity mode only: it places one D2H job per offloaded
// layer at that layer's production time on the simulated bus. On the device
// the same per-layer jobs are issued by lkv_prefill_layer().
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "layersim/cost_model.hpp"
#include "layersim/interconnect.hpp"

namespace layersim {

struct PrefillSchedule {
  double completion = 0.0;
  std::vector<TransferSchedule> jobs;
};

PrefillSchedule schedule_prefill_span(const ModelSpec& model, const HardwareSpec& hw,
                                      const CostParams& cost, PcieBus& bus,
                                      std::span<const int> offloaded_layers,
                                      std::int64_t prompt_tokens, double start,
                                      double chunk_bytes, bool transfers_enabled);

}  // namespace layersim
