"""Prefill softmax / MMA phase trace (development aid; needs a library built
with -DLKV_PREFILL_TRACE=1, scripts/build_variant.sh trace ...).

  python scripts/prefill_trace.py --lib build/variants/trace/liblkv.so [--tokens 16384]

CTA 0 (the heaviest query-tile pair) stamps clock64 per KV tile j: softmax
warp of each tile (S ready, S in registers, row max, P computed, P stored) and
the MMA warp (loop top, PV_A+S_A issued, PV_B+S_B issued). Prints the median
phase lengths in cycles over the steady-state tiles."""
import argparse
import ctypes as C
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2410_00428_b200 import _abi  # noqa: E402
from paper_2410_00428_b200 import layersim as ls  # noqa: E402
from paper_2410_00428_b200.device import DTYPE_BF16, Device, DeviceConfig  # noqa: E402


def cta_timeline(lib, n_ctas, items_per_pair_tiles):
    """Per-CTA %globaltimer spans (start, end, SM) of the last launch."""
    buf = (C.c_ulonglong * (3 * 4096))()
    assert lib.dll.lkv_debug_prefill_cta(buf, 3 * 4096) == 0
    rows = [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(min(n_ctas, 4096))]
    t0 = min(r[0] for r in rows)
    t1 = max(r[1] for r in rows)
    busy = {}
    for a, b, smid in rows:
        busy[smid] = busy.get(smid, 0) + (b - a)
    span = t1 - t0
    durs = sorted(b - a for a, b, _ in rows)
    return {"ctas": len(rows), "span_us": span / 1e3, "sm_busy_frac": sum(busy.values()) / (len(busy) * span),
            "sms": len(busy), "cta_us_min_med_max": [durs[0] / 1e3, durs[len(durs) // 2] / 1e3, durs[-1] / 1e3],
            "last_start_us": (max(r[0] for r in rows) - t0) / 1e3}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--lib", required=True)
    p.add_argument("--tokens", type=int, default=16384)
    p.add_argument("--hq", type=int, default=32)
    p.add_argument("--hkv", type=int, default=8)
    a = p.parse_args()
    lib = _abi.Lib(a.lib)
    model = ls.ModelSpec(1, a.hq, a.hkv, 128, a.hq * 128, 8e9, 2)
    kv = ls.KvManager(ls.BlockPools(64, 64, 16), model, lib=lib)
    dev = Device(kv, model, 16, DeviceConfig(gpu_slots=64, host_slots=64, arena_slots=64, max_requests=2,
                                             max_blocks=64, max_batch=2), lib=lib)
    T = a.tokens
    q = (torch.rand((T, a.hq, 128), device="cuda") * 2 - 1).to(torch.bfloat16)
    k = (torch.rand((T, a.hkv, 128), device="cuda") * 2 - 1).to(torch.bfloat16)
    v = (torch.rand((T, a.hkv, 128), device="cuda") * 2 - 1).to(torch.bfloat16)
    out = torch.empty_like(q)
    for _ in range(3):
        dev.prefill_attention(q, k, v, out, T, 1 / math.sqrt(128), DTYPE_BF16)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 4096)()
    assert lib.dll.lkv_debug_prefill_trace(buf, 4096) == 0
    tr = list(buf)
    nt = (T + 127) // 128  # CTA 0 = heaviest pair: tiles 0 .. nq-1
    res = {"tokens": T}
    names = ["s_ready", "s_in_regs", "max_done", "p_computed", "p_stored"]
    for t in (0, 1):
        ph = {f"{names[i]}->{names[i + 1]}": [] for i in range(4)}
        ph["p_stored->next_s_ready"] = []
        for j in range(4, min(nt - 2, 127)):
            b = t * 1024 + j * 8
            for i in range(4):
                ph[f"{names[i]}->{names[i + 1]}"].append(tr[b + i + 1] - tr[b + i])
            ph["p_stored->next_s_ready"].append(tr[b + 8] - tr[b + 4])
        res[f"tile_{'AB'[t]}"] = {kk: statistics.median(vv) for kk, vv in ph.items() if vv}
    mm = {"top->pvA_sA_issued": [], "pvA_sA->pvB_issued": [], "period": [], "wait_v": [], "wait_k": [],
          "pvB_issued->next_loop": []}
    for j in range(4, min(nt - 2, 127)):
        b = 2048 + j * 8
        mm["top->pvA_sA_issued"].append(tr[b + 1] - tr[b])
        mm["pvA_sA->pvB_issued"].append(tr[b + 2] - tr[b + 1])
        mm["period"].append(tr[b + 8] - tr[b])
        mm["wait_v"].append(tr[b + 8 + 4] - tr[b + 8 + 3])
        mm["wait_k"].append(tr[b + 8] - tr[b + 8 + 4])
        mm["pvB_issued->next_loop"].append(tr[b + 8 + 3] - tr[b + 2])
    res["mma_warp"] = {kk: statistics.median(vv) for kk, vv in mm.items()}
    res["softmax_A_vs_mma"] = "cycles (clock64, one SM)"
    nq = (T + 127) // 128
    res["timeline"] = cta_timeline(lib, ((nq + 1) // 2) * a.hq, None)
    print(json.dumps(res))
    dev.close()


if __name__ == "__main__":
    main()
