"""TEST INFRASTRUCTURE — the oracles for the LayerKV path.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this package, and only as the checker / the timed CPU reference; the
product (paper_2410_00428_b200) never imports it.

* ``ref_lib()``     the reference C++ sources compiled in place
                    (oracle/_ref/libref_layersim.so, built here by
                    ``make -C oracle ref``; needs /root/reference, so on the
                    GPU box it exists only if built before the snapshot).
* ``hybrid_lib()``  reference engine.cpp linked with the product
                    KvManager/PcieBus/cost model (drop-in proof).
* ``restatement()`` CPU restatement in C (kvgen.c, attn_ref.c): synthetic KV
                    generator + fp32 paged decode attention. Builds anywhere
                    gcc exists (also on the GPU box).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libref_layersim.so")
HYB_SO = os.path.join(HERE, "_ref", "libhybrid_layersim.so")
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REFERENCE_SRC = "/root/reference/proj"


def build(ref: bool = True) -> None:
    """Build the restatement always; the reference shims when its sources exist."""
    targets = ["restatement"]
    if ref and os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO) and os.path.exists(HYB_SO)


def _load_abi(path):
    import sys
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_2410_00428_b200 import _abi
    lib = _abi.Lib(path, device=False)
    lib.dll.ref_engine_run.restype = C.c_int32
    lib.dll.ref_generate_trace.restype = C.c_int32
    lib.dll.ref_generate_trace.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_uint64,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    return lib


_cache = {}


def ref_lib():
    if "ref" not in _cache:
        if not os.path.exists(REF_SO):
            build()
        _cache["ref"] = _load_abi(REF_SO)
    return _cache["ref"]


def hybrid_lib():
    if "hyb" not in _cache:
        if not os.path.exists(HYB_SO):
            build()
        _cache["hyb"] = _load_abi(HYB_SO)
    return _cache["hyb"]


class Restatement:
    def __init__(self, path):
        d = C.CDLL(path)
        d.oracle_kv_value_bf16.restype = C.c_uint16
        d.oracle_kv_value_bf16.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int]
        d.oracle_q_value_bf16.restype = C.c_uint16
        d.oracle_q_value_bf16.argtypes = [C.c_uint64, C.c_int, C.c_int64, C.c_int, C.c_int]
        d.oracle_fill_kv.restype = None
        d.oracle_fill_kv.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                                     C.c_int, C.c_uint64]
        d.oracle_slot_bytes.restype = None
        d.oracle_slot_bytes.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_int64, C.c_uint64]
        d.oracle_decode_attn.restype = None
        d.oracle_decode_attn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                         C.c_int, C.c_float, C.c_void_p]
        d.oracle_decode_attn_gen.restype = None
        d.oracle_decode_attn_gen.argtypes = [C.c_uint64, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.c_void_p, C.c_float, C.c_void_p]
        d.oracle_prefill_attn.restype = None
        d.oracle_prefill_attn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int,
                                          C.c_float, C.c_void_p]
        self.dll = d

    # numpy helpers -------------------------------------------------------
    def fill_kv(self, tokens, token0, layer, heads, head0, dim, seed):
        import numpy as np
        k = np.empty((tokens, heads, dim), np.uint16)
        v = np.empty_like(k)
        self.dll.oracle_fill_kv(k.ctypes.data, v.ctypes.data, tokens, token0, layer, heads, head0, dim, seed)
        return k, v

    def slot_bytes(self, layer, block, bs, heads, head0, dim, n_tokens, seed):
        import numpy as np
        out = np.empty((2, heads, bs, dim), np.uint16)
        self.dll.oracle_slot_bytes(out.ctypes.data, layer, block, bs, heads, head0, dim, n_tokens, seed)
        return out

    def q_values(self, seed, layer, n_seq, hq_local, head0_q, dim):
        import numpy as np
        q = np.empty((n_seq, hq_local, dim), np.uint16)
        for s in range(n_seq):
            for h in range(hq_local):
                for d in range(dim):
                    q[s, h, d] = self.dll.oracle_q_value_bf16(seed, layer, s, head0_q + h, d)
        return q

    def decode_attn(self, q, k, v, scale):
        import numpy as np
        q = np.ascontiguousarray(q, np.uint16)
        k = np.ascontiguousarray(k, np.uint16)
        v = np.ascontiguousarray(v, np.uint16)
        hq, d = q.shape
        kv_len, hkv, _ = k.shape
        out = np.empty((hq, d), np.float32)
        self.dll.oracle_decode_attn(q.ctypes.data, k.ctypes.data, v.ctypes.data, kv_len, hq, hkv, d, scale,
                                    out.ctypes.data)
        return out

    def prefill_attn(self, q, k, v, scale):
        """Causal attention, q [T][hq][d], k/v [T][hkv][d] (bf16 bits) -> fp32 [T][hq][d]."""
        import numpy as np
        q = np.ascontiguousarray(q, np.uint16)
        k = np.ascontiguousarray(k, np.uint16)
        v = np.ascontiguousarray(v, np.uint16)
        T, hq, d = q.shape
        out = np.empty((T, hq, d), np.float32)
        self.dll.oracle_prefill_attn(q.ctypes.data, k.ctypes.data, v.ctypes.data, T, hq, k.shape[1], d, scale,
                                     out.ctypes.data)
        return out

    def decode_attn_gen(self, seed, layer, kv_len, head0, hkv_local, group, q, scale):
        import numpy as np
        q = np.ascontiguousarray(q, np.uint16)
        out = np.empty((hkv_local * group, q.shape[-1]), np.float32)
        self.dll.oracle_decode_attn_gen(seed, layer, kv_len, head0, hkv_local, group, q.shape[-1], q.ctypes.data,
                                        scale, out.ctypes.data)
        return out


def restatement() -> Restatement:
    if "re" not in _cache:
        if not os.path.exists(ORACLE_SO):
            subprocess.run(["make", "-s", "-C", HERE, "restatement"], check=True)
        _cache["re"] = Restatement(ORACLE_SO)
    return _cache["re"]
