// Parity-mode per-layer offload schedule (reference engine.cpp:22-45): layer l
// ends at start + (l+1) * T/L; an offloaded layer submits its whole-prompt
// D2H job at that instant; the span itself always completes at start + T.
#include "layersim/prefill_span.hpp"

namespace layersim {

PrefillSchedule schedule_prefill_span(const ModelSpec& model, const HardwareSpec& hw,
                                      const CostParams& cost, PcieBus& bus,
                                      std::span<const int> offloaded, std::int64_t prompt,
                                      double start, double chunk_bytes, bool enabled) {
  const double T = prefill_time(model, hw, cost, prompt);
  const double per_layer = T / model.n_layers;
  const double ar = allreduce_time(model, hw, prompt);
  const double layer_bytes =
      static_cast<double>(prompt) * static_cast<double>(kv_bytes_per_token_layer(model));
  PrefillSchedule out;
  out.completion = start + T;
  std::size_t next = 0;
  for (int l = 0; l < model.n_layers; ++l) {
    const double end = start + (l + 1) * per_layer;
    if (ar > 0.0) bus.register_allreduce(end - ar, ar, hw);
    if (!enabled || next >= offloaded.size() || offloaded[next] != l) continue;
    out.jobs.push_back(
        bus.submit_transfer({layer_bytes, Direction::DeviceToHost, end, chunk_bytes}, hw));
    ++next;
  }
  return out;
}

}  // namespace layersim
