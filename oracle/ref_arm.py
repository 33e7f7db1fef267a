"""TEST INFRASTRUCTURE — the CPU reference arm of bench.py. Never shipped.

Used only by ``bench.py --impl reference`` and by bench.py's ``cpu_baseline``
leg; it does not import the product package (``paper_2410_00428_b200``), so
the reference arm loads no product library.

* ``RefKvManager``: the REFERENCE KvManager (proj/src/kv_manager.cpp, compiled
  in place into oracle/_ref/libref_layersim.so by oracle/Makefile) through its
  C shim (oracle/ref_shim.cpp), with a minimal ctypes binding of its own:
  allocate_prefill, the request's block table, plan_decode_fetch.
* ``ref_simulated_ttft``: the reference Engine::run (engine.cpp:76-121, the
  same compiled library) over the reference's own generate_fixed trace —
  config 2's simulated TTFT p50/p99 as the reference computes it, timed on
  one host core (the reference is single-threaded).
* ``Port``: the oracle CPU port of one decode step (oracle/cpu_baseline.c):
  per (request, layer) it gathers the layer's slots from host frames into a
  contiguous arena with memcpy (the fetch the reference books,
  kv_manager.cpp:290-304) and runs fp32 paged attention over it, on all host
  threads. One arena per Port, touched once, so both bench legs time the same
  code over the same kind of memory.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import time

import numpy as np

from . import REF_SO, restatement

i32, i64, u8, u32, f64 = C.c_int32, C.c_int64, C.c_uint8, C.c_uint32, C.c_double


class _ModelSpec(C.Structure):  # include/lkv.h lkv_model_spec
    _fields_ = [("n_layers", i32), ("n_heads", i32), ("n_kv_heads", i32), ("d_head", i32),
                ("hidden", i64), ("n_param", f64), ("f_precision", i32), ("pad_", i32)]


class _BlockPools(C.Structure):  # lkv_block_pools
    _fields_ = [("gpu_blocks_total", i64), ("cpu_blocks_total", i64), ("tokens_per_block", i32), ("pad_", i32)]


class _SlotLoc(C.Structure):  # lkv_slot_loc
    _fields_ = [("loc", u8), ("offload_in_flight", u8), ("pad_", C.c_uint16), ("slot", u32), ("dest_slot", u32)]


class _FetchJob(C.Structure):  # lkv_fetch_job
    _fields_ = [("layer", i32), ("pad_", i32), ("bytes", f64)]


LLAMA2_7B = (32, 32, 32, 128, 4096, 7.0e9, 2)  # reference config.cpp model_preset("llama2-7b")


def kv_bytes_per_token_layer(model=LLAMA2_7B) -> int:
    """reference cost_model.cpp kv_bytes_per_token_layer: 2 (K, V) x Hkv x d x f."""
    return 2 * model[2] * model[3] * model[6]


class _HardwareSpec(C.Structure):  # lkv_hardware_spec
    _fields_ = [("flops", f64), ("hbm_bandwidth", f64), ("pcie_bandwidth", f64), ("nvlink", i32), ("n_gpus", i32),
                ("gpu_mem", f64), ("kv_reserve_fraction", f64)]


class _CostParams(C.Structure):  # lkv_cost_params
    _fields_ = [("alpha", f64), ("beta", f64), ("gamma", f64), ("delta", f64)]


class _EngineCfg(C.Structure):  # oracle/ref_shim.cpp ref_engine_cfg
    _fields_ = [("model", _ModelSpec), ("hw", _HardwareSpec), ("cost", _CostParams), ("ttft_slo", f64),
                ("tpot_slo", f64), ("policy_layerkv", i32), ("slo_scheduler", i32), ("gpu_blocks", i64),
                ("cpu_blocks", i64), ("tokens_per_block", i32), ("horizon", i32), ("threshold_fraction", f64),
                ("predictor_accuracy", f64), ("max_batch_tokens", i64), ("max_sim_time", f64),
                ("chunk_bytes", f64), ("seed", C.c_uint64), ("force_retained_layers", i32),
                ("invariant_checks", i32)]


class _EngineOut(C.Structure):  # ref_engine_out
    _fields_ = [("mean_ttft", f64), ("p50_ttft", f64), ("p99_ttft", f64), ("mean_tpot", f64), ("throughput", f64),
                ("makespan", f64), ("d2h_jobs", i64), ("h2d_jobs", i64), ("d2h_bytes", f64), ("h2d_bytes", f64),
                ("completed", i32), ("n_rows", i32)]


def ref_simulated_ttft(ctx: int, n: int = 100, output: int = 512, rate: float = 1.0, seed: int = 1) -> dict:
    """Config 2: generate_fixed(n, ctx, output, rate, seed)
    through the reference Engine::run with the reference defaults
    (config.cpp: L20-like HardwareSpec 1e14 / 8.64e11 / 3.2e10, 48 GB, cost
    params 1/1/1/0.5, SLOs 3 s / 0.2 s, horizon 8) and the 48 GB-capped
    pools 113,043 / 904,344; both policies. Host time on one core."""
    if not os.path.exists(REF_SO):
        raise RuntimeError(f"reference library not built: {REF_SO} (make -C oracle ref)")
    dll = C.CDLL(REF_SO)
    dll.ref_engine_run.restype = i32
    dll.ref_generate_trace.restype = i32
    dll.lkv_last_error.restype = C.c_char_p
    ids, arr = (i64 * n)(), (f64 * n)()
    p, o = (i32 * n)(), (i32 * n)()
    if dll.ref_generate_trace(0, n, ctx, output, C.c_double(rate), C.c_uint64(seed), ids, arr, p, o) != 0:
        raise RuntimeError("ref_generate_trace failed")
    out = {"unit": "s", "source": "compiled reference Engine::run (oracle/_ref), virtual time"}
    for pol in ("layerkv", "baseline"):
        cfg = _EngineCfg(_ModelSpec(*LLAMA2_7B, 0), _HardwareSpec(1.0e14, 8.64e11, 3.2e10, 0, 1, 48e9, 0.9),
                         _CostParams(1.0, 1.0, 1.0, 0.5), 3.0, 0.2, int(pol == "layerkv"), 1, 113043, 904344, 16, 8,
                         0.05, 0.8, 131072, 86400.0, 16.0 * 1024 * 1024, seed, -1, 0)
        res = _EngineOut()
        ln = C.c_size_t()
        t0 = time.perf_counter()
        st = dll.ref_engine_run(C.byref(cfg), n, ids, arr, p, o, C.byref(res), None, C.c_size_t(0), C.byref(ln))
        host_s = time.perf_counter() - t0
        if st != 0:
            raise RuntimeError("ref_engine_run: " + dll.lkv_last_error().decode())
        out[pol] = {"p50": res.p50_ttft, "p99": res.p99_ttft, "mean_tpot": res.mean_tpot,
                    "tokens_per_s": res.throughput, "host_s_1core": host_s}
    return out


class RefKvManager:
    def __init__(self, gpu_blocks, cpu_blocks, bs, model=LLAMA2_7B):
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"reference library not built: {REF_SO} (make -C oracle ref)")
        d = C.CDLL(REF_SO, mode=C.RTLD_LOCAL)
        for name in ("lkv_kv_create", "lkv_kv_destroy", "lkv_kv_allocate_prefill", "lkv_kv_request_shape",
                     "lkv_kv_request_table", "lkv_kv_plan_decode_fetch"):
            getattr(d, name).restype = i32
        d.lkv_last_error.restype = C.c_char_p
        self.dll, self.model, self.bs = d, model, bs
        self.h = C.c_void_p()
        self._ok(d.lkv_kv_create(C.byref(_BlockPools(gpu_blocks, cpu_blocks, bs, 0)), C.byref(_ModelSpec(*model, 0)),
                                 C.byref(self.h)))

    def _ok(self, st):
        if st != 0:
            raise RuntimeError(self.dll.lkv_last_error().decode(errors="replace"))

    def close(self):
        if self.h:
            self.dll.lkv_kv_destroy(self.h)
            self.h = None

    def allocate_prefill(self, rid, tokens, x) -> bool:
        ok = i32()
        self._ok(self.dll.lkv_kv_allocate_prefill(self.h, i64(rid), i64(tokens), i32(x), C.byref(ok)))
        return bool(ok.value)

    def slots(self, rid):
        """[layer][block] slot ids of the request (block table, kv_manager.hpp RequestKv)."""
        cached, nb = i64(), i64()
        self._ok(self.dll.lkv_kv_request_shape(self.h, i64(rid), C.byref(cached), C.byref(nb)))
        L = self.model[0]
        ent = (_SlotLoc * (nb.value * L))()
        self._ok(self.dll.lkv_kv_request_table(self.h, i64(rid), ent, None, None))
        return [[ent[b * L + l].slot for b in range(nb.value)] for l in range(L)]

    def plan_decode_fetch(self, rid):
        n = i32()
        self._ok(self.dll.lkv_kv_plan_decode_fetch(self.h, i64(rid), None, 0, C.byref(n)))
        out = (_FetchJob * max(1, n.value))()
        self._ok(self.dll.lkv_kv_plan_decode_fetch(self.h, i64(rid), out, n.value, C.byref(n)))
        return [(out[i].layer, out[i].bytes) for i in range(n.value)]


class Port:
    """oracle/cpu_baseline.c cpu_decode_layer with one pre-touched arena."""

    def __init__(self, nblk, slot_bytes, kv_len, hkv, group, bs, d, threads=None):
        fn = restatement().dll.cpu_decode_layer
        fn.restype = None
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                       C.c_void_p, C.c_float, C.c_void_p, C.c_void_p, C.c_int]
        self.fn = fn
        self.threads = threads or os.cpu_count() or 1
        self.shape = (nblk, slot_bytes, kv_len, hkv, group, bs, d)
        self.arena = np.zeros(nblk * slot_bytes, np.uint8)  # touched once, reused by every call
        q = np.random.default_rng(0).random((hkv * group, d), dtype=np.float32) * 2 - 1
        self.q16 = (q.view(np.uint32) >> 16).astype(np.uint16)
        self.out = np.empty((hkv * group, d), np.float32)
        self.scale = 1.0 / math.sqrt(d)

    def layer(self, host_pool_ptr, slots: np.ndarray):
        nblk, slot_bytes, kv_len, hkv, group, bs, d = self.shape
        self.fn(host_pool_ptr, slots.ctypes.data, nblk, slot_bytes, kv_len, hkv, group, bs, d, self.q16.ctypes.data,
                self.scale, self.out.ctypes.data, self.arena.ctypes.data, self.threads)

    def kv_bytes(self, layers: int) -> int:
        nblk, slot_bytes, kv_len, hkv, group, bs, d = self.shape
        return layers * kv_len * 2 * hkv * d * 2

    def timed(self, host_pool_ptr, slots_per_layer, seconds):
        """Whole passes over the given (request, layer) slot lists until `seconds` are spent.
        Returns (GB/s of KV consumed, layers done, elapsed s)."""
        rows = [np.asarray(s, np.uint32) for s in slots_per_layer]
        t0 = time.perf_counter()
        done = 0
        while True:
            for s in rows:
                self.layer(host_pool_ptr, s)
                done += 1
            if time.perf_counter() - t0 > seconds:
                break
        dt = time.perf_counter() - t0
        return self.kv_bytes(done) / dt / 1e9, done, dt
