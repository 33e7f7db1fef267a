"""Serving loop and trace formats over the C ABI.

Mirrors the reference's caller of the path: ``EngineConfig`` / ``Engine.run``
(engine.hpp:32-80), ``generate_fixed`` / ``generate_sharegpt_like`` /
``load_trace`` / ``save_trace`` (workload.hpp) and ``requests.csv``
(metrics.cpp:91-101). The executor picks the time source:

* ``"modelled"``        cost model + serial PcieBus: the reference's numbers;
* ``"device-virtual"``  the GPU executes every job, the clock stays modelled;
* ``"device-measured"`` the GPU executes and CUDA events are the clock.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import _abi
from .layersim import CostParams, HardwareSpec, ModelSpec, default_hardware

EXECUTORS = {"modelled": 0, "device-virtual": 1, "device-measured": 2}


@dataclass
class Trace:
    """reference workload.hpp:17-22 (requests sorted by arrival)."""
    ids: list
    arrival: list
    prompt: list
    output: list

    def __len__(self):
        return len(self.ids)

    def arrays(self):
        n = len(self.ids)
        return ((C.c_int64 * n)(*self.ids), (C.c_double * n)(*self.arrival), (C.c_int32 * n)(*self.prompt),
                (C.c_int32 * n)(*self.output))


@dataclass
class ServeConfig:
    """reference EngineConfig (engine.hpp:32-50) + the device executor's knobs."""
    model: ModelSpec
    hw: HardwareSpec = field(default_factory=default_hardware)
    cost: CostParams = field(default_factory=CostParams)
    ttft_slo: float = 3.0
    tpot_slo: float = 0.2
    layerkv: bool = True
    slo_scheduler: bool = True
    gpu_blocks: int = 0
    cpu_blocks: int = 0
    tokens_per_block: int = 16
    horizon: int = 8
    threshold_fraction: float = 0.05
    predictor_accuracy: float = 0.8
    max_batch_tokens: int = 131072
    max_time: float = 86400.0
    chunk_bytes: float = 16.0 * 1024 * 1024
    seed: int = 0
    force_retained_layers: int = -1
    invariant_checks: bool = False
    executor: str = "modelled"
    device: int = 0
    dense_gemms: bool = True
    prefill_attention: bool = True
    verify_kv: bool = False
    pipeline_depth: int = 2
    ffn: int = 0
    host_slots: int = 0
    kv_seed: int = 0x4C61796572
    tp_rank: int = 0  # the KV-head shard the device executes; tp_size = hw.n_gpus
    pinned_frames: int = 0  # > 0: the f3 tier (pageable homes, this many pinned frames)

    def c(self) -> _abi.ServeConfigC:
        return _abi.ServeConfigC(
            self.model.c(), self.hw.c(), self.cost.c(), self.ttft_slo, self.tpot_slo, int(self.layerkv),
            int(self.slo_scheduler), self.gpu_blocks, self.cpu_blocks, self.tokens_per_block, self.horizon,
            self.threshold_fraction, self.predictor_accuracy, self.max_batch_tokens, self.max_time, self.chunk_bytes,
            self.seed, self.force_retained_layers, int(self.invariant_checks), EXECUTORS[self.executor], self.device,
            int(self.dense_gemms), int(self.prefill_attention), int(self.verify_kv), self.pipeline_depth, self.ffn,
            self.host_slots, self.kv_seed, self.tp_rank, 0, self.pinned_frames)


def _lib(lib=None):
    return lib or _abi.product_lib()


def generate_fixed(n: int, prompt: int, output: int, rate: float, seed: int, lib=None) -> Trace:
    return _generate(False, n, prompt, output, rate, seed, lib)


def generate_sharegpt_like(n: int, rate: float, seed: int, lib=None) -> Trace:
    return _generate(True, n, 0, 0, rate, seed, lib)


def _generate(sharegpt, n, prompt, output, rate, seed, lib):
    ids, arr, p, o = (C.c_int64 * n)(), (C.c_double * n)(), (C.c_int32 * n)(), (C.c_int32 * n)()
    _lib(lib).call("lkv_trace_generate", int(sharegpt), n, prompt, output, rate, seed, ids, arr, p, o)
    return Trace(list(ids), list(arr), list(p), list(o))


def load_trace(path: str, lib=None):
    """Returns (trace, was_unsorted)."""
    L = _lib(lib)
    n, uns = C.c_int32(), C.c_int32()
    L.call("lkv_trace_read_jsonl", str(path).encode(), None, None, None, None, 0, C.byref(n), C.byref(uns))
    k = n.value
    ids, arr, p, o = (C.c_int64 * k)(), (C.c_double * k)(), (C.c_int32 * k)(), (C.c_int32 * k)()
    L.call("lkv_trace_read_jsonl", str(path).encode(), ids, arr, p, o, k, C.byref(n), C.byref(uns))
    return Trace(list(ids), list(arr), list(p), list(o)), bool(uns.value)


def save_trace(trace: Trace, path: str, lib=None):
    _lib(lib).call("lkv_trace_write_jsonl", str(path).encode(), len(trace), *trace.arrays())


def requests_csv(rows, lib=None) -> str:
    L = _lib(lib)
    n = len(rows)
    arr = (_abi.ServeRowC * max(n, 1))(*rows)
    ln = C.c_size_t()
    L.call("lkv_serve_requests_csv", arr, n, None, 0, C.byref(ln))
    buf = C.create_string_buffer(ln.value + 1)
    L.call("lkv_serve_requests_csv", arr, n, buf, ln.value + 1, C.byref(ln))
    return buf.raw[:ln.value].decode()


def run(cfg: ServeConfig, trace: Trace, lib=None, logs=False):
    """Engine::run. Returns (summary dict, rows, requests.csv text), and with
    logs=True also the run's transfer_log.csv and decision_log.csv texts (the
    reference CLI's --transfer-log / --decision-log files,
    tools/layersim_main.cpp:96-117)."""
    L = _lib(lib)
    n = len(trace)
    out = _abi.ServeSummaryC()
    rows = (_abi.ServeRowC * n)()
    if not logs:
        L.call("lkv_serve_run", C.byref(cfg.c()), n, *trace.arrays(), C.byref(out), rows, n)
    else:
        cap, dcap = 1 << 20, 1 << 16
        while True:  # the logs' sizes are known only after the run: rerun once with room for them
            buf, ln = C.create_string_buffer(cap), C.c_size_t()
            dbuf, dln = C.create_string_buffer(dcap), C.c_size_t()
            L.call("lkv_serve_run_ex", C.byref(cfg.c()), n, *trace.arrays(), C.byref(out), rows, n, buf, cap,
                   C.byref(ln), dbuf, dcap, C.byref(dln))
            if ln.value < cap and dln.value < dcap:
                break
            cap, dcap = max(cap, ln.value + 1), max(dcap, dln.value + 1)
    summary = {k: getattr(out, k) for k, _ in out._fields_ if k != "pad_"}
    got = list(rows)[:out.n_rows]
    if logs:
        return summary, got, requests_csv(got, L), buf.raw[:ln.value].decode(), dbuf.raw[:dln.value].decode()
    return summary, got, requests_csv(got, L)
