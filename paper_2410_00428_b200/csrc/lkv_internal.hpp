// Internal glue shared by the C-ABI translation units.
#pragma once

#include <stdexcept>
#include <string>

#include "layersim/cost_model.hpp"
#include "layersim/kv_manager.hpp"
#include "lkv.h"

namespace lkv {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
struct CapacityError : std::runtime_error {
  explicit CapacityError(const std::string& m) : std::runtime_error(m) {}
};

void set_error(const std::string& msg);
int status_from_current_exception();
layersim::ModelSpec to_model(const lkv_model_spec* m);
layersim::KvManager& kv_impl(lkv_kv_manager* kv);
// device.cu: bind a device to a manager owned elsewhere (the serving loop).
void device_bind_manager(lkv_device* d, layersim::KvManager& k);

}  // namespace lkv
