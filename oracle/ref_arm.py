"""TEST INFRASTRUCTURE — the CPU reference arm of bench.py. Never shipped.

Used only by ``bench.py --impl reference`` and by bench.py's ``cpu_baseline``
leg; it does not import the product package (``paper_2410_00428_b200``), so
the reference arm loads no product library.

* ``RefKvManager``: the REFERENCE KvManager (proj/src/kv_manager.cpp, compiled
  in place into oracle/_ref/libref_layersim.so by oracle/Makefile) through its
  C shim (oracle/ref_shim.cpp), with a minimal ctypes binding of its own:
  allocate_prefill, the request's block table, plan_decode_fetch.
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
