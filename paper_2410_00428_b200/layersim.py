"""Python mirror of the reference's C++ API for the LayerKV path.

Same names, argument meaning and error behaviour as the reference headers
(proj/include/layersim/{cost_model,kv_manager,interconnect,engine}.hpp):
capacity failures are return values (False / None), logic errors raise
SimulationError / ConfigError / DomainError / InvalidArgument. Every call goes
through the C ABI (include/lkv.h) of a loaded library; by default the product
library, in parity tests optionally the reference shim.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _abi
from ._abi import (ConfigError, DomainError, InvalidArgument, SimulationError, CapacityError,  # noqa: F401
                   CudaError, LkvError)

HALF, FULL = 0, 1
LOC_NONE, LOC_GPU, LOC_CPU = 0, 1, 2
D2H, H2D = 0, 1


# --------------------------------------------------------------------- specs
@dataclass
class ModelSpec:
    """reference cost_model.hpp:9-19."""
    n_layers: int = 0
    n_heads: int = 0
    n_kv_heads: int = 0
    d_head: int = 0
    hidden: int = 0
    n_param: float = 0.0
    f_precision: int = 0

    def c(self) -> _abi.ModelSpec:
        return _abi.ModelSpec(self.n_layers, self.n_heads, self.n_kv_heads, self.d_head, self.hidden,
                              self.n_param, self.f_precision, 0)


@dataclass
class HardwareSpec:
    """reference cost_model.hpp:21-31."""
    flops: float = 0.0
    hbm_bandwidth: float = 0.0
    pcie_bandwidth: float = 0.0
    nvlink: bool = False
    n_gpus: int = 1
    gpu_mem: float = 0.0
    kv_reserve_fraction: float = 0.9

    def c(self) -> _abi.HardwareSpec:
        return _abi.HardwareSpec(self.flops, self.hbm_bandwidth, self.pcie_bandwidth, int(self.nvlink),
                                 self.n_gpus, self.gpu_mem, self.kv_reserve_fraction)


@dataclass
class CostParams:
    alpha: float = 1.0
    beta: float = 1.0
    gamma: float = 1.0
    delta: float = 0.5

    def c(self) -> _abi.CostParams:
        return _abi.CostParams(self.alpha, self.beta, self.gamma, self.delta)


@dataclass
class PoolSizing:
    max_input_tokens: int = 16384
    tokens_per_block: int = 16
    activation_layers_factor: float = 4.0
    cpu_pool_multiple: float = 8.0


@dataclass
class BlockPools:
    gpu_blocks_total: int = 0
    cpu_blocks_total: int = 0
    tokens_per_block: int = 16


@dataclass
class OffloadJob:
    job_id: int = -1
    request_id: int = -1
    bytes: float = 0.0
    layer_count: int = 0
    gpu_blocks: int = 0


@dataclass
class FetchJob:
    layer: int = 0
    bytes: float = 0.0


@dataclass
class FreedCounts:
    gpu: int = 0
    cpu: int = 0
    deferred_gpu: int = 0


@dataclass
class SlotLoc:
    loc: int = LOC_NONE
    slot: int = 0
    offload_in_flight: bool = False
    dest_slot: int = 0


@dataclass
class LogicalBlock:
    token_begin: int = 0
    layers: List[SlotLoc] = field(default_factory=list)


@dataclass
class RequestKv:
    id: int = -1
    cached_tokens: int = 0
    blocks: List[LogicalBlock] = field(default_factory=list)
    layer_residency: List[int] = field(default_factory=list)


@dataclass
class PlacementPlan:
    retained: List[int]
    offloaded: List[int]


@dataclass
class TransferSchedule:
    start: float = 0.0
    completion: float = 0.0
    chunks: int = 0
    deferrals: int = 0


# presets the reference tests and configs use (reference config.cpp:146-171)
def llama2_7b() -> ModelSpec:
    return ModelSpec(32, 32, 32, 128, 4096, 7.0e9, 2)


def llama3_8b_gqa() -> ModelSpec:
    return ModelSpec(32, 32, 8, 128, 4096, 8.03e9, 2)


def llama31_70b_gqa() -> ModelSpec:
    return ModelSpec(80, 64, 8, 128, 8192, 70.6e9, 2)


def tiny8() -> ModelSpec:
    return ModelSpec(8, 4, 4, 32, 128, 1e8, 2)


def default_hardware() -> HardwareSpec:
    return HardwareSpec(1.0e14, 8.64e11, 3.2e10, False, 1, 48e9, 0.9)


def _lib(lib):
    return lib if lib is not None else _abi.product_lib()


# ------------------------------------------------------------ cost model
def kv_bytes_per_token_layer(m: ModelSpec, lib=None) -> int:
    out = C.c_int64()
    _lib(lib).call("lkv_kv_bytes_per_token_layer", C.byref(m.c()), C.byref(out))
    return out.value


def prefill_time(m: ModelSpec, hw: HardwareSpec, p: CostParams, seqlen: int, lib=None) -> float:
    out = C.c_double()
    _lib(lib).call("lkv_prefill_time", C.byref(m.c()), C.byref(hw.c()), C.byref(p.c()), seqlen, C.byref(out))
    return out.value


def offload_time(m, hw, p, seqlen: int, layers_offloaded: int, lib=None) -> float:
    out = C.c_double()
    _lib(lib).call("lkv_offload_time", C.byref(m.c()), C.byref(hw.c()), C.byref(p.c()), seqlen,
                   layers_offloaded, C.byref(out))
    return out.value


def min_retained_layers(m, hw, p, seqlen: int, lib=None) -> int:
    out = C.c_int32()
    _lib(lib).call("lkv_min_retained_layers", C.byref(m.c()), C.byref(hw.c()), C.byref(p.c()), seqlen,
                   C.byref(out))
    return out.value


def decode_step_time(m, hw, p, batch_kv_tokens: int, lib=None) -> float:
    out = C.c_double()
    _lib(lib).call("lkv_decode_step_time", C.byref(m.c()), C.byref(hw.c()), C.byref(p.c()), batch_kv_tokens,
                   C.byref(out))
    return out.value


def allreduce_time(m, hw, tokens: int, lib=None) -> float:
    out = C.c_double()
    _lib(lib).call("lkv_allreduce_time", C.byref(m.c()), C.byref(hw.c()), tokens, C.byref(out))
    return out.value


def pool_size_from_hardware(m: ModelSpec, hw: HardwareSpec, s: PoolSizing, lib=None) -> BlockPools:
    out = _abi.BlockPools()
    cs = _abi.PoolSizing(s.max_input_tokens, s.tokens_per_block, 0, s.activation_layers_factor,
                         s.cpu_pool_multiple)
    _lib(lib).call("lkv_pool_size_from_hardware", C.byref(m.c()), C.byref(hw.c()), C.byref(cs), C.byref(out))
    return BlockPools(out.gpu_blocks_total, out.cpu_blocks_total, out.tokens_per_block)


def layer_placement(n_layers: int, x: int, lib=None) -> PlacementPlan:
    ret = (C.c_int32 * max(x, 1))()
    off = (C.c_int32 * max(n_layers - x, 1))()
    _lib(lib).call("lkv_layer_placement", n_layers, x, ret, off)
    return PlacementPlan(list(ret[:x]), list(off[:n_layers - x]))


# ------------------------------------------------------------ KvManager
class KvManager:
    """Drop-in mirror of layersim::KvManager (reference kv_manager.hpp:80-150)."""

    def __init__(self, pools: BlockPools, model: ModelSpec, lib=None):
        self._lib = _lib(lib)
        self.model = model
        h = C.c_void_p()
        self._lib.call("lkv_kv_create", C.byref(_abi.BlockPools(pools.gpu_blocks_total, pools.cpu_blocks_total,
                                                                 pools.tokens_per_block, 0)),
                       C.byref(model.c()), C.byref(h))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self._lib.dll.lkv_kv_destroy(h)
            self.handle = None

    def _i64(self, name, *args) -> int:
        out = C.c_int64()
        self._lib.call(name, self.handle, *args, C.byref(out))
        return out.value

    def _i32(self, name, *args) -> int:
        out = C.c_int32()
        self._lib.call(name, self.handle, *args, C.byref(out))
        return out.value

    def stats(self) -> _abi.KvStats:
        s = _abi.KvStats()
        self._lib.call("lkv_kv_stats_get", self.handle, C.byref(s))
        return s

    def tokens_per_block(self) -> int:
        return self.stats().tokens_per_block

    def gpu_blocks_total(self) -> int:
        return self.stats().gpu_blocks_total

    def gpu_blocks_free(self) -> int:
        return self.stats().gpu_blocks_free

    def cpu_blocks_total(self) -> int:
        return self.stats().cpu_blocks_total

    def cpu_blocks_free(self) -> int:
        return self.stats().cpu_blocks_free

    def blocks_per_layer(self, tokens: int) -> int:
        return self._i64("lkv_kv_blocks_per_layer", tokens)

    def request_wise_gpu_blocks(self, prompt_tokens: int) -> int:
        return self._i64("lkv_kv_request_wise_gpu_blocks", prompt_tokens)

    def allocate_prefill(self, request_id: int, prompt_tokens: int, x: int) -> bool:
        return bool(self._i32("lkv_kv_allocate_prefill", request_id, prompt_tokens, x))

    def has_request(self, request_id: int) -> bool:
        return bool(self._i32("lkv_kv_has_request", request_id))

    def request(self, request_id: int) -> RequestKv:
        cached, nb = C.c_int64(), C.c_int64()
        self._lib.call("lkv_kv_request_shape", self.handle, request_id, C.byref(cached), C.byref(nb))
        L = self.model.n_layers
        ent = (_abi.SlotLocC * max(1, nb.value * L))()
        tb = (C.c_int64 * max(1, nb.value))()
        res = (C.c_uint8 * L)()
        self._lib.call("lkv_kv_request_table", self.handle, request_id, ent, tb, res)
        blocks = []
        for b in range(nb.value):
            row = [SlotLoc(e.loc, e.slot, bool(e.offload_in_flight), e.dest_slot) for e in ent[b * L:(b + 1) * L]]
            blocks.append(LogicalBlock(tb[b], row))
        return RequestKv(request_id, cached.value, blocks, list(res))

    def request_table_raw(self, request_id: int):
        """(cached_tokens, entries ctypes array [b*L+l]) — fast path for tests."""
        cached, nb = C.c_int64(), C.c_int64()
        self._lib.call("lkv_kv_request_shape", self.handle, request_id, C.byref(cached), C.byref(nb))
        ent = (_abi.SlotLocC * max(1, nb.value * self.model.n_layers))()
        self._lib.call("lkv_kv_request_table", self.handle, request_id, ent, None, None)
        return cached.value, nb.value, ent

    def retained_layer_count(self, request_id: int) -> int:
        return self._i32("lkv_kv_retained_layer_count", request_id)

    def gpu_blocks_held(self, request_id: int) -> int:
        return self._i64("lkv_kv_gpu_blocks_held", request_id)

    def gpu_row_cost(self, request_id: int) -> int:
        return self._i64("lkv_kv_gpu_row_cost", request_id)

    def cpu_row_cost(self, request_id: int) -> int:
        return self._i64("lkv_kv_cpu_row_cost", request_id)

    def offload_reclaim(self, request_id: int, mode: int) -> int:
        return self._i64("lkv_kv_offload_reclaim", request_id, mode)

    def plan_offload(self, request_id: int, mode: int) -> Optional[OffloadJob]:
        job, has = _abi.OffloadJobC(), C.c_int32()
        self._lib.call("lkv_kv_plan_offload", self.handle, request_id, mode, C.byref(job), C.byref(has))
        if not has.value:
            return None
        return OffloadJob(job.job_id, job.request_id, job.bytes, job.layer_count, job.gpu_blocks)

    def complete_offload(self, job_id: int) -> None:
        self._lib.call("lkv_kv_complete_offload", self.handle, job_id)

    def plan_decode_fetch(self, request_id: int) -> List[FetchJob]:
        n = C.c_int32()
        self._lib.call("lkv_kv_plan_decode_fetch", self.handle, request_id, None, 0, C.byref(n))
        buf = (_abi.FetchJobC * max(1, n.value))()
        self._lib.call("lkv_kv_plan_decode_fetch", self.handle, request_id, buf, n.value, C.byref(n))
        return [FetchJob(j.layer, j.bytes) for j in buf[:n.value]]

    def needs_append(self, request_id: int) -> bool:
        return bool(self._i32("lkv_kv_needs_append", request_id))

    def append_decode_block(self, request_id: int) -> bool:
        return bool(self._i32("lkv_kv_append_decode_block", request_id))

    def note_token(self, request_id: int) -> None:
        self._lib.call("lkv_kv_note_token", self.handle, request_id)

    def release(self, request_id: int) -> FreedCounts:
        f = _abi.FreedCountsC()
        self._lib.call("lkv_kv_release", self.handle, request_id, C.byref(f))
        return FreedCounts(f.gpu, f.cpu, f.deferred_gpu)

    def check_conservation(self) -> None:
        self._lib.call("lkv_kv_check_conservation", self.handle)

    def dump_table(self) -> str:
        n = C.c_size_t()
        self._lib.call("lkv_kv_dump_table", self.handle, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        self._lib.call("lkv_kv_dump_table", self.handle, buf, n.value + 1, C.byref(n))
        return buf.raw[:n.value].decode()

    def free_stack(self, gpu: bool = True):
        """The LIFO free list as the reference's SlotPool keeps it
        (kv_manager.hpp:153-166): bottom to top, next allocation last."""
        n = C.c_int64()
        which = 0 if gpu else 1
        self._lib.call("lkv_kv_free_stack", self.handle, which, None, 0, C.byref(n))
        out = (C.c_uint32 * max(1, n.value))()
        self._lib.call("lkv_kv_free_stack", self.handle, which, out, n.value, C.byref(n))
        return list(out)[:n.value]

    def free_delta(self, gpu: bool = True, full: bool = False):
        """The free-list journal the device mirror applies (include/lkv.h
        lkv_kv_free_delta): (next_fresh, low, size, changed, pushed[low:size])."""
        nf, lo, sz, ch = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
        cap = self.gpu_blocks_total() if gpu else self.cpu_blocks_total()
        out = (C.c_uint32 * max(1, cap))()
        self._lib.call("lkv_kv_free_delta", self.handle, 0 if gpu else 1, 1 if full else 0, C.byref(nf), C.byref(lo),
                       C.byref(sz), C.byref(ch), out, cap)
        return nf.value, lo.value, sz.value, bool(ch.value), list(out)[:sz.value - lo.value]

    def dump_hash(self) -> int:
        h = C.c_uint64()
        self._lib.call("lkv_kv_dump_hash", self.handle, C.byref(h))
        return h.value


# ------------------------------------------------------------ PcieBus
class PcieBus:
    """Parity-mode host-link timing (reference interconnect.hpp:45-73)."""

    def __init__(self, delta: float = 0.5, lib=None):
        self._lib = _lib(lib)
        h = C.c_void_p()
        self._lib.call("lkv_bus_create", delta, C.byref(h))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self._lib.dll.lkv_bus_destroy(h)
            self.handle = None

    def register_allreduce(self, start: float, duration: float, hw: HardwareSpec) -> None:
        self._lib.call("lkv_bus_register_allreduce", self.handle, start, duration, C.byref(hw.c()))

    def submit_transfer(self, bytes_: float, direction: int, submit_time: float, chunk_bytes: float,
                        hw: HardwareSpec) -> TransferSchedule:
        s = _abi.TransferScheduleC()
        self._lib.call("lkv_bus_submit_transfer", self.handle, bytes_, direction, submit_time, chunk_bytes,
                       C.byref(hw.c()), C.byref(s))
        return TransferSchedule(s.start, s.completion, s.chunks, s.deferrals)

    def _state(self, t=0.0):
        a, b, c = C.c_double(), C.c_double(), C.c_int32()
        self._lib.call("lkv_bus_state", self.handle, t, C.byref(a), C.byref(b), C.byref(c))
        return a.value, b.value, bool(c.value)

    def busy_until(self) -> float:
        return self._state()[0]

    def allreduce_busy_until(self) -> float:
        return self._state()[1]

    def allreduce_active(self, t: float) -> bool:
        return self._state(t)[2]

    def enable_history(self, on: bool) -> None:
        self._lib.call("lkv_bus_enable_history", self.handle, int(on))

    def _spans(self, name):
        n = C.c_int32()
        self._lib.call(name, self.handle, None, 0, C.byref(n))
        buf = (_abi.SpanC * max(1, n.value))()
        self._lib.call(name, self.handle, buf, n.value, C.byref(n))
        return [(s.begin, s.end, bool(s.is_allreduce)) for s in buf[:n.value]]

    def chunk_history(self):
        return self._spans("lkv_bus_chunk_history")

    def allreduce_windows(self):
        return self._spans("lkv_bus_allreduce_windows")


def schedule_prefill_span(m: ModelSpec, hw: HardwareSpec, p: CostParams, bus: PcieBus,
                          offloaded_layers: Sequence[int], prompt_tokens: int, start: float,
                          chunk_bytes: float, transfers_enabled: bool, lib=None):
    """reference engine.hpp:67-71; returns (completion, [TransferSchedule])."""
    lib = _lib(lib)
    off = (C.c_int32 * max(1, len(offloaded_layers)))(*offloaded_layers)
    comp, n = C.c_double(), C.c_int32()
    jobs = (_abi.TransferScheduleC * max(1, m.n_layers))()
    lib.call("lkv_schedule_prefill_span", C.byref(m.c()), C.byref(hw.c()), C.byref(p.c()), bus.handle, off,
             len(offloaded_layers), prompt_tokens, start, chunk_bytes, int(transfers_enabled), C.byref(comp),
             jobs, m.n_layers, C.byref(n))
    return comp.value, [TransferSchedule(j.start, j.completion, j.chunks, j.deferrals) for j in jobs[:n.value]]
