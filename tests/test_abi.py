"""The C-ABI library loads and exports every entry point include/lkv.h declares
(no compute calls; runs without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "lkv.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"LKV_API\s+(?:const\s+)?\w+\*?\s+\**(lkv_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    assert len(syms) >= 60
    for must in ("lkv_kv_allocate_prefill", "lkv_kv_plan_offload", "lkv_kv_complete_offload",
                 "lkv_kv_plan_decode_fetch", "lkv_bus_submit_transfer", "lkv_schedule_prefill_span",
                 "lkv_prefill_layer", "lkv_decode_begin", "lkv_decode_layer", "lkv_device_bind"):
        assert must in syms


def test_product_library_exports_every_declared_symbol(prod):
    dll = ctypes.CDLL(prod.path)
    missing = [s for s in declared_symbols() if not hasattr(dll, s)]
    assert not missing, missing
    assert prod.version().endswith("sm_100a")


def test_product_library_is_sm100a_code():
    import subprocess
    so = os.path.join(ROOT, "paper_2410_00428_b200", "liblkv.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_python_binding_covers_header(prod):
    from paper_2410_00428_b200 import _abi
    assert set(declared_symbols()) <= set(_abi.ALL_SYMBOLS)


def test_reference_shim_exports_bookkeeping_half(ref):
    from paper_2410_00428_b200 import _abi
    dll = ctypes.CDLL(ref.path)
    book = [s for s in declared_symbols() if s not in _abi.DEVICE_SYMBOLS]
    assert all(hasattr(dll, s) for s in book)
