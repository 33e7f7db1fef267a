"""Config-5 sweep (BASELINE.json configs[4]): offload / prefetch bandwidth of
the device path over layers offloaded, block size, context and KV-head shard.

Each point: one request of `ctx` tokens, allocate_prefill with x = L - k
retained layers, per-layer prefill through lkv_prefill_layer (pack kernel +
D2H copy engine into the CPU slots' pinned frames) timed end to end, then one
decode iteration (H2D prefetch of the k offloaded layers, layer-ahead, plus
paged attention) timed with the device's CUDA events. Shards: TP = N runs
rank 0's KV-head shard on this GPU (per-GPU bytes = total / N; every GPU has
its own link and copy engines). GB/s are algorithmic bytes over copy-engine
busy time (CUDA events around each batch of copies); the wall-clock view of
the prefill path and the prefetch span are reported beside them. One JSON
line per point.

  python scripts/sweep_offload.py [--quick] > sweep.jsonl
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

SEED = 0x4C61796572


def link_peak():
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        out[name] = 3 * n / (time.perf_counter() - t0) / 1e9
    return out


def point(model, label, tp, bs, ctx, k, peak):
    L = model.n_layers
    x = L - k
    nblk = (ctx + bs - 1) // bs
    kv = ls.KvManager(ls.BlockPools(nblk * L + 64, nblk * L + 64, bs), model)
    dev = Device(kv, model, bs, DeviceConfig(tp_rank=0, tp_size=tp, gpu_slots=nblk * x + 64, host_slots=nblk * k + 64,
                                             arena_slots=nblk + 16, max_requests=2, max_blocks=nblk + 8,
                                             max_batch=1, staging_chunks=16, chunk_bytes=16 << 20))
    dev.set_timing(True)
    hl, hq = dev.kv_heads_local, dev.q_heads_local
    kk = torch.empty((ctx, hl, 128), dtype=torch.bfloat16, device="cuda")
    vv = torch.empty_like(kk)
    cs = dev.torch_stream()
    dev.fill_kv(kk, vv, ctx, 0, 0, SEED, stream=cs)
    assert kv.allocate_prefill(0, ctx, x)
    dev.synchronize()
    dev.offload_stats(reset=True)
    t0 = time.perf_counter()
    for layer in range(L):
        dev.prefill_layer(0, layer, kk, vv, ctx, stream=cs)
    dev.synchronize()
    t_off = time.perf_counter() - t0
    ost = dev.offload_stats(reset=True)
    q = torch.randn((1, hq, 128), dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(q)
    best = None
    for it in range(2):
        dev.decode_begin([0])
        for layer in range(L):
            dev.decode_layer(layer, q, out, 1 / math.sqrt(128), DTYPE_BF16, stream=cs)
        dev.decode_end()
        st = dev.decode_stats()
        if best is None or st.iteration_ms < best.iteration_ms:
            best = st
    dev.close()
    h2d_gbs = best.h2d_bytes_algorithmic / (best.h2d_ms / 1e3) / 1e9 if best.h2d_ms else None  # copy-busy
    d2h_gbs = ost.d2h_bytes_algorithmic / (ost.d2h_ms / 1e3) / 1e9 if ost.d2h_ms else None  # copy-busy
    return {"model": label, "tp": tp, "bs": bs, "ctx": ctx, "layers_offloaded": k, "layers": L,
            "offload_bytes_per_gpu": ost.d2h_bytes_algorithmic,
            "offload_gbs_per_gpu": d2h_gbs, "offload_frac_of_d2h_peak": d2h_gbs / peak["d2h"] if d2h_gbs else None,
            "offload_gbs_prefill_wall": ost.d2h_bytes_algorithmic / t_off / 1e9,
            "offload_copies": ost.d2h_copies, "prefill_path_ms": t_off * 1e3,
            "prefetch_bytes_per_gpu": best.h2d_bytes_algorithmic, "prefetch_gbs_per_gpu": h2d_gbs,
            "prefetch_frac_of_h2d_peak": h2d_gbs / peak["h2d"] if h2d_gbs else None,
            "prefetch_copies": best.h2d_copies, "decode_iteration_ms": best.iteration_ms,
            "prefetch_gbs_span": best.h2d_bytes_algorithmic / (best.h2d_span_ms / 1e3) / 1e9 if best.h2d_span_ms else None,
            "attn_ms": best.attn_ms}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--quick", action="store_true")
    a = p.parse_args()
    peak = link_peak()
    print(json.dumps({"link_peak_gbs": peak}), flush=True)
    m7 = ls.llama2_7b()
    m70 = ls.llama31_70b_gqa()
    pts = []
    for bs in (16, 32, 64):  # block size: DMA / gather granularity only (job bytes are bs-independent)
        pts.append((m7, "llama2-7b", 1, bs, 16384, 16))
    for ctx in (4096, 16384, 65536, 131072):
        pts.append((m7, "llama2-7b", 1, 16, ctx, 1 if ctx > 65536 else 4))
    for k in (1, 8, 32):
        pts.append((m7, "llama2-7b", 1, 16, 8192, k))
    for tp in (1, 2, 4, 8):  # config 4: 70B GQA sharded by KV head, half of 80 layers offloaded
        pts.append((m70, "llama3.1-70b-gqa", tp, 16, 8192, 40))
    pts.append((m70, "llama3.1-70b-gqa", 8, 16, 131072, 40))
    pts.append((m70, "llama3.1-70b-gqa", 8, 64, 131072, 80))
    if a.quick:
        pts = pts[:3]
    for args in pts:
        r = point(*args, peak)
        print(json.dumps(r), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
