"""ctypes binding of include/lkv.h.

This is the binding a maintainer of the reference would add to reach the C
ABI from Python. The same binding drives two libraries with
identical symbols: the product ``liblkv.so`` (this package) and, in tests
only, the reference shim ``oracle/_ref/libref_layersim.so``.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblkv.so")

i32, i64, u8, u32, u64, f64, f32 = C.c_int32, C.c_int64, C.c_uint8, C.c_uint32, C.c_uint64, C.c_double, C.c_float
P = C.POINTER
vp = C.c_void_p
IPC_HANDLE_BYTES = 64  # LKV_IPC_HANDLE_BYTES (cudaIpcMemHandle_t)


class ModelSpec(C.Structure):
    _fields_ = [("n_layers", i32), ("n_heads", i32), ("n_kv_heads", i32), ("d_head", i32),
                ("hidden", i64), ("n_param", f64), ("f_precision", i32), ("pad_", i32)]


class HardwareSpec(C.Structure):
    _fields_ = [("flops", f64), ("hbm_bandwidth", f64), ("pcie_bandwidth", f64),
                ("nvlink", i32), ("n_gpus", i32), ("gpu_mem", f64), ("kv_reserve_fraction", f64)]


class CostParams(C.Structure):
    _fields_ = [("alpha", f64), ("beta", f64), ("gamma", f64), ("delta", f64)]


class PoolSizing(C.Structure):
    _fields_ = [("max_input_tokens", i64), ("tokens_per_block", i32), ("pad_", i32),
                ("activation_layers_factor", f64), ("cpu_pool_multiple", f64)]


class BlockPools(C.Structure):
    _fields_ = [("gpu_blocks_total", i64), ("cpu_blocks_total", i64),
                ("tokens_per_block", i32), ("pad_", i32)]


class OffloadJobC(C.Structure):
    _fields_ = [("job_id", i64), ("request_id", i64), ("bytes", f64), ("layer_count", i32),
                ("pad_", i32), ("gpu_blocks", i64)]


class FetchJobC(C.Structure):
    _fields_ = [("layer", i32), ("pad_", i32), ("bytes", f64)]


class FreedCountsC(C.Structure):
    _fields_ = [("gpu", i64), ("cpu", i64), ("deferred_gpu", i64)]


class SlotLocC(C.Structure):
    _fields_ = [("loc", u8), ("offload_in_flight", u8), ("pad_", C.c_uint16), ("slot", u32),
                ("dest_slot", u32)]


class KvStats(C.Structure):
    _fields_ = [("gpu_blocks_total", i64), ("gpu_blocks_free", i64), ("cpu_blocks_total", i64),
                ("cpu_blocks_free", i64), ("tokens_per_block", i32), ("n_layers", i32),
                ("pending_offloads", i64), ("live_requests", i64)]


class TransferScheduleC(C.Structure):
    _fields_ = [("start", f64), ("completion", f64), ("chunks", i32), ("deferrals", i32)]


class SpanC(C.Structure):
    _fields_ = [("begin", f64), ("end", f64), ("is_allreduce", i32), ("pad_", i32)]


class ServeConfigC(C.Structure):
    _fields_ = [("model", ModelSpec), ("hw", HardwareSpec), ("cost", CostParams), ("ttft_slo", f64),
                ("tpot_slo", f64), ("policy_layerkv", i32), ("slo_scheduler", i32), ("gpu_blocks", i64),
                ("cpu_blocks", i64), ("tokens_per_block", i32), ("horizon", i32), ("threshold_fraction", f64),
                ("predictor_accuracy", f64), ("max_batch_tokens", i64), ("max_time", f64), ("chunk_bytes", f64),
                ("seed", u64), ("force_retained_layers", i32), ("invariant_checks", i32), ("executor", i32),
                ("device", i32), ("dense_gemms", i32), ("prefill_attention", i32), ("verify_kv", i32),
                ("pipeline_depth", i32), ("ffn", i64), ("host_slots", i64), ("kv_seed", u64), ("tp_rank", i32), ("pad_", i32),
                ("pinned_frames", i64)]


class ServeSummaryC(C.Structure):
    _fields_ = [("mean_ttft", f64), ("p50_ttft", f64), ("p99_ttft", f64), ("mean_tpot", f64), ("throughput", f64),
                ("makespan", f64), ("d2h_jobs", i64), ("h2d_jobs", i64), ("d2h_bytes", f64), ("h2d_bytes", f64),
                ("completed", i32), ("n_rows", i32), ("violations", i32), ("pad_", i32), ("prefills", i64),
                ("decode_iterations", i64), ("kv_words_mismatched", i64), ("requests_verified", i64),
                ("gpu_kernel_launches", i64), ("prefill_device_s", f64), ("decode_device_s", f64), ("escalations", i64)]


class ServeRowC(C.Structure):
    _fields_ = [("id", i64), ("arrival", f64), ("queuing", f64), ("prefill", f64), ("ttft", f64),
                ("mean_tpot", f64), ("output_tokens", i32), ("violated", i32)]


class DeviceConfig(C.Structure):
    _fields_ = [("device", i32), ("tp_rank", i32), ("tp_size", i32), ("pipeline_depth", i32),
                ("gpu_slots", i64), ("host_slots", i64), ("arena_slots", i64),
                ("max_requests", i32), ("max_blocks", i32), ("max_batch", i32),
                ("staging_chunks", i32), ("chunk_bytes", i64), ("pinned_frames", i64)]


class HostTierStats(C.Structure):
    _fields_ = [("pinned_frames", i64), ("read_in_frames", i64), ("write_back_frames", i64), ("evictions", i64),
                ("hits", i64), ("misses", i64), ("staged", i64), ("pin_waits", i64), ("read_ahead", i32),
                ("copy_threads", i32), ("resident_frames", i64)]


class DeviceInfo(C.Structure):
    _fields_ = [("slot_bytes", i64), ("kv_heads_local", i32), ("q_heads_local", i32),
                ("head_dim", i32), ("tokens_per_block", i32), ("pool", vp), ("host_pool", vp),
                ("arena", vp), ("compute_stream", vp), ("d2h_stream", vp), ("h2d_stream", vp),
                ("numa_node", i32), ("gather_peers", i32)]


class DecodeStats(C.Structure):
    _fields_ = [("h2d_bytes_physical", i64), ("h2d_bytes_algorithmic", i64), ("h2d_copies", i64),
                ("kv_bytes_read", i64), ("attn_launches", i64), ("kernel_launches", i64), ("attn_ms", f64),
                ("h2d_ms", f64),
                ("iteration_ms", f64), ("h2d_span_ms", f64), ("merge_ms", f64), ("kernel_ms", f64)]


class OffloadStats(C.Structure):
    _fields_ = [("d2h_bytes_physical", i64), ("d2h_bytes_algorithmic", i64), ("d2h_copies", i64),
                ("jobs", i64), ("scatter_bytes", i64), ("d2h_ms", f64), ("pack_ms", f64),
                ("scatter_ms", f64)]


# name -> (argtypes); every function returns int32 status unless listed in _RET
_PROTOS = {
    "lkv_model_validate": [P(ModelSpec)],
    "lkv_kv_bytes_per_token_layer": [P(ModelSpec), P(i64)],
    "lkv_prefill_time": [P(ModelSpec), P(HardwareSpec), P(CostParams), i64, P(f64)],
    "lkv_offload_time": [P(ModelSpec), P(HardwareSpec), P(CostParams), i64, i32, P(f64)],
    "lkv_min_retained_layers": [P(ModelSpec), P(HardwareSpec), P(CostParams), i64, P(i32)],
    "lkv_decode_step_time": [P(ModelSpec), P(HardwareSpec), P(CostParams), i64, P(f64)],
    "lkv_allreduce_time": [P(ModelSpec), P(HardwareSpec), i64, P(f64)],
    "lkv_pool_size_from_hardware": [P(ModelSpec), P(HardwareSpec), P(PoolSizing), P(BlockPools)],
    "lkv_layer_placement": [i32, i32, P(i32), P(i32)],
    "lkv_kv_create": [P(BlockPools), P(ModelSpec), P(vp)],
    "lkv_kv_destroy": [vp],
    "lkv_kv_stats_get": [vp, P(KvStats)],
    "lkv_kv_blocks_per_layer": [vp, i64, P(i64)],
    "lkv_kv_request_wise_gpu_blocks": [vp, i64, P(i64)],
    "lkv_kv_allocate_prefill": [vp, i64, i64, i32, P(i32)],
    "lkv_kv_has_request": [vp, i64, P(i32)],
    "lkv_kv_request_shape": [vp, i64, P(i64), P(i64)],
    "lkv_kv_request_table": [vp, i64, P(SlotLocC), P(i64), P(u8)],
    "lkv_kv_retained_layer_count": [vp, i64, P(i32)],
    "lkv_kv_gpu_blocks_held": [vp, i64, P(i64)],
    "lkv_kv_gpu_row_cost": [vp, i64, P(i64)],
    "lkv_kv_cpu_row_cost": [vp, i64, P(i64)],
    "lkv_kv_offload_reclaim": [vp, i64, i32, P(i64)],
    "lkv_kv_plan_offload": [vp, i64, i32, P(OffloadJobC), P(i32)],
    "lkv_kv_complete_offload": [vp, i64],
    "lkv_kv_plan_decode_fetch": [vp, i64, P(FetchJobC), i32, P(i32)],
    "lkv_kv_needs_append": [vp, i64, P(i32)],
    "lkv_kv_append_decode_block": [vp, i64, P(i32)],
    "lkv_kv_note_token": [vp, i64],
    "lkv_kv_release": [vp, i64, P(FreedCountsC)],
    "lkv_kv_check_conservation": [vp],
    "lkv_kv_dump_table": [vp, C.c_char_p, C.c_size_t, P(C.c_size_t)],
    "lkv_kv_dump_hash": [vp, P(u64)],
    "lkv_kv_free_stack": [vp, i32, P(u32), i64, P(i64)],
    "lkv_device_numa_node": [i32, P(i32)],
    "lkv_kv_free_delta": [vp, i32, i32, P(i64), P(i64), P(i64), P(i32), P(u32), i64],
    "lkv_bus_create": [f64, P(vp)],
    "lkv_bus_destroy": [vp],
    "lkv_bus_register_allreduce": [vp, f64, f64, P(HardwareSpec)],
    "lkv_bus_submit_transfer": [vp, f64, i32, f64, f64, P(HardwareSpec), P(TransferScheduleC)],
    "lkv_bus_state": [vp, f64, P(f64), P(f64), P(i32)],
    "lkv_bus_enable_history": [vp, i32],
    "lkv_bus_chunk_history": [vp, P(SpanC), i32, P(i32)],
    "lkv_bus_allreduce_windows": [vp, P(SpanC), i32, P(i32)],
    "lkv_schedule_prefill_span": [P(ModelSpec), P(HardwareSpec), P(CostParams), vp, P(i32), i32,
                                  i64, f64, f64, i32, P(f64), P(TransferScheduleC), i32, P(i32)],
    # device half (absent from the reference shim)
    "lkv_device_create": [P(ModelSpec), i32, P(DeviceConfig), P(vp)],
    "lkv_device_destroy": [vp],
    "lkv_device_get_info": [vp, P(DeviceInfo)],
    "lkv_device_bind": [vp, vp],
    "lkv_device_synchronize": [vp],
    "lkv_prefill_layer": [vp, i64, i32, vp, vp, i64, vp],
    "lkv_prefill_attention": [vp, vp, vp, vp, vp, i64, f32, i32, vp],
    "lkv_device_job_done": [vp, i64, P(i32)],
    "lkv_device_prefill_offload_done": [vp, i64, P(i32)],
    "lkv_decode_begin": [vp, P(i64), i32],
    "lkv_decode_layer": [vp, i32, vp, vp, f32, i32, vp],
    "lkv_decode_begin_append": [vp, P(i64), i32],
    "lkv_decode_append_layer": [vp, i32, vp, vp, vp],
    "lkv_decode_end": [vp],
    "lkv_device_gather_ipc_handle": [vp, vp],
    "lkv_device_gather_connect_ipc": [vp, vp, i32],
    "lkv_device_gather_buffer": [vp, P(vp), P(u64)],
    "lkv_device_gather_connect": [vp, P(vp), i32],
    "lkv_decode_gather_wait": [vp, i32, vp],
    "lkv_decode_gathered": [vp, i32, P(vp)],
    "lkv_device_set_timing": [vp, i32],
    "lkv_decode_last_stats": [vp, P(DecodeStats)],
    "lkv_offload_last_stats": [vp, P(OffloadStats), i32],
    "lkv_fill_kv": [vp, vp, vp, i64, i64, i32, u64, vp],
    "lkv_fill_kv_tokens": [vp, vp, vp, P(i64), i32, i32, u64, vp],
    # serving loop and trace formats
    "lkv_serve_run": [P(ServeConfigC), i32, P(i64), P(f64), P(i32), P(i32), P(ServeSummaryC), P(ServeRowC), i32],
    "lkv_serve_run_ex": [P(ServeConfigC), i32, P(i64), P(f64), P(i32), P(i32), P(ServeSummaryC), P(ServeRowC), i32,
                         C.c_char_p, C.c_size_t, P(C.c_size_t), C.c_char_p, C.c_size_t, P(C.c_size_t)],
    "lkv_serve_requests_csv": [P(ServeRowC), i32, C.c_char_p, C.c_size_t, P(C.c_size_t)],
    "lkv_trace_generate": [i32, i32, i32, i32, f64, u64, P(i64), P(f64), P(i32), P(i32)],
    "lkv_trace_read_jsonl": [C.c_char_p, P(i64), P(f64), P(i32), P(i32), i32, P(i32), P(i32)],
    "lkv_trace_write_jsonl": [C.c_char_p, i32, P(i64), P(f64), P(i32), P(i32)],
    "lkv_verify_request": [vp, i64, i64, u64, P(i64)],
    "lkv_fill_request": [vp, i64, i64, u64],
    "lkv_device_read_host_slot": [vp, i64, vp],
    "lkv_device_free_stack": [vp, i32, P(u32), i64, P(i64)],
    "lkv_device_host_tier_stats": [vp, P(HostTierStats)],
}
_RET = {"lkv_last_error": C.c_char_p, "lkv_version": C.c_char_p}

DEVICE_SYMBOLS = [n for n in _PROTOS if n.startswith(("lkv_device", "lkv_prefill_layer", "lkv_prefill_attention", "lkv_decode_begin",
                                                     "lkv_decode_layer", "lkv_decode_end", "lkv_decode_last",
                                                     "lkv_decode_append", "lkv_decode_gather",
                                                     "lkv_offload_last", "lkv_fill", "lkv_verify",
                                                     "lkv_serve", "lkv_trace"))]
ALL_SYMBOLS = list(_PROTOS) + list(_RET)


class LkvError(RuntimeError):
    """Base of the status-code exceptions."""


class SimulationError(LkvError):
    """layersim::SimulationError (reference errors.hpp:14-17)."""


class ConfigError(LkvError):
    """layersim::ConfigError (reference errors.hpp:9-12)."""


class DomainError(LkvError, ValueError):
    """std::domain_error."""


class InvalidArgument(LkvError, ValueError):
    """std::invalid_argument / bad C argument."""


class CudaError(LkvError):
    pass


class CapacityError(LkvError):
    pass


_STATUS = {-1: SimulationError, -2: ConfigError, -3: DomainError, -4: InvalidArgument,
           -5: CudaError, -6: CapacityError, -7: LkvError}


class Lib:
    """A loaded library exposing the lkv C ABI (product or reference shim)."""

    def __init__(self, path: str, device: bool = True):
        if not os.path.exists(path):
            raise ImportError(f"lkv C-ABI library not built: {path} (run __graft_entry__.build())")
        self.path = path
        self.dll = C.CDLL(path, mode=C.RTLD_LOCAL)
        self.has_device = device
        for name, args in _PROTOS.items():
            fn = getattr(self.dll, name, None)
            if fn is None:
                if not device and name in DEVICE_SYMBOLS:
                    continue
                raise ImportError(f"{path}: missing symbol {name}")
            fn.argtypes = args
            fn.restype = i32
        for name, ret in _RET.items():
            fn = getattr(self.dll, name)
            fn.argtypes = []
            fn.restype = ret

    def call(self, name: str, *args):
        st = getattr(self.dll, name)(*args)
        if st != 0:
            msg = self.dll.lkv_last_error().decode(errors="replace")
            raise _STATUS.get(st, LkvError)(f"{name}: {msg}")
        return st

    def version(self) -> str:
        return self.dll.lkv_version().decode()


_PRODUCT: Lib | None = None


def product_lib() -> Lib:
    """The product library. Fails loudly when the extension is missing —
    there is no CPU fallback for the device path."""
    global _PRODUCT
    if _PRODUCT is None:
        _PRODUCT = Lib(LIB_PATH, device=True)
    return _PRODUCT
