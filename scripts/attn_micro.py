"""Decode-attention microbenchmark (development aid; the judged numbers come
from bench.py). Same shape as the bench step (7 x 16k tokens, 7B), but with
every layer GPU-resident so only the attention kernel is timed.

  python scripts/attn_micro.py [--group 1] [--ctx 16384] [--batch 7] [--layers 4]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2410_00428_b200 import layersim as ls  # noqa: E402
from paper_2410_00428_b200.device import DTYPE_BF16, Device, DeviceConfig  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--group", type=int, default=1)
    p.add_argument("--hkv", type=int, default=0)
    p.add_argument("--ctx", type=int, default=16384)
    p.add_argument("--batch", type=int, default=7)
    p.add_argument("--layers", type=int, default=4)
    p.add_argument("--bs", type=int, default=16)
    p.add_argument("--iters", type=int, default=5)
    p.add_argument("--offloaded", action="store_true", help="every layer CPU-resident: per-layer H2D prefetch "
                   "runs beside the kernels, as in the bench step")
    p.add_argument("--idle-ms", type=float, default=0.0, help="leave the GPU idle this long before each layer")
    p.add_argument("--lib", default=None, help="an alternative liblkv.so (scripts/build_variant.sh)")
    p.add_argument("--label", default="default")
    a = p.parse_args()
    from paper_2410_00428_b200 import _abi
    lib = _abi.Lib(a.lib) if a.lib else None
    hkv = a.hkv or (32 if a.group == 1 else 8)
    model = ls.ModelSpec(a.layers, hkv * a.group, hkv, 128, hkv * a.group * 128, 7e9, 2)
    nblk = (a.ctx + a.bs - 1) // a.bs
    slots = a.batch * nblk * a.layers
    gslots, hslots = (64, slots + 64) if a.offloaded else (slots + 64, 64)
    kv = ls.KvManager(ls.BlockPools(gslots, hslots, a.bs), model, lib=lib)
    cfg = DeviceConfig(gpu_slots=gslots, host_slots=hslots, arena_slots=a.batch * nblk + 8, max_requests=a.batch + 1,
                       max_blocks=nblk + 4, max_batch=a.batch, pipeline_depth=2)
    dev = Device(kv, model, a.bs, cfg, lib=lib)
    ids = list(range(a.batch))
    for r in ids:
        assert kv.allocate_prefill(r, a.ctx, 0 if a.offloaded else a.layers)
        dev.fill_request(r, a.ctx, 1)
    hq = dev.q_heads_local
    q = torch.randn((a.batch, hq, 128), dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(q)
    dev.set_timing(True)
    res, kres, kspan = [], [], []
    for it in range(a.iters + 2):
        dev.decode_begin(ids)
        for l in range(a.layers):
            if a.idle_ms:
                dev.synchronize()
                time.sleep(a.idle_ms / 1e3)
            dev.decode_layer(l, q, out, 1 / math.sqrt(128), DTYPE_BF16)
        dev.decode_end()
        st = dev.decode_stats()
        if it >= 2:
            res.append((st.attn_ms + st.merge_ms) / st.attn_launches)
            kspan.append(st.kernel_ms / st.attn_launches)
            kres.append(st.attn_ms / st.attn_launches)
    kvb = a.batch * a.ctx * 2 * hkv * 128 * 2
    ms = min(res)
    print(json.dumps({"variant": a.label,
                      "offloaded": a.offloaded, "idle_ms": a.idle_ms, "merge_ms": ms - min(kres),
                      "group": a.group, "hkv": hkv, "batch": a.batch, "ctx": a.ctx, "bs": a.bs,
                      "ms_per_layer": ms, "kernel_ms": min(kres), "kernel_ms_mean": sum(kres) / len(kres), "kernel_span_ms": min(kspan), "GBps": kvb / (ms / 1e3) / 1e9,
                      "kernel_frac_of_6536.7": kvb / (min(kres) / 1e3) / 1e9 / 6536.7,
                      "frac_of_6536.7": kvb / (ms / 1e3) / 1e9 / 6536.7}))
    dev.close()


if __name__ == "__main__":
    main()
