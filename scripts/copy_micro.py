"""Data-movement kernel microbenchmark (development aid): the scatter of a
retained prefill layer into its GPU slots, the pack of an offloaded layer
into staging, and the escalation gather of GPU slots into staging, on the
7B shape (32 KV heads, bs 16, 256 KiB slots), through the C ABI.

  python scripts/copy_micro.py [--tokens 16384] [--layers 4]

Prints CUDA-event times of lkv_prefill_layer (scatter or pack + D2H enqueue)
and algorithmic HBM GB/s (read K/V + write slots). Run under
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`
for per-kernel numbers.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2410_00428_b200 import layersim as ls  # noqa: E402
from paper_2410_00428_b200.device import Device, DeviceConfig  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--tokens", type=int, default=16384)
    p.add_argument("--layers", type=int, default=4)
    a = p.parse_args()
    T, L, bs = a.tokens, a.layers, 16
    model = ls.ModelSpec(L, 32, 32, 128, 4096, 7e9, 2)
    nblk = T // bs
    kv = ls.KvManager(ls.BlockPools(nblk * L + 64, nblk * L + 64, bs), model)
    dev = Device(kv, model, bs, DeviceConfig(gpu_slots=nblk * L + 64, host_slots=nblk * L + 64, arena_slots=64,
                                             max_requests=4, max_blocks=nblk + 4, max_batch=2, staging_chunks=64,
                                             chunk_bytes=16 << 20))
    cs = dev.torch_stream("compute")
    k = torch.empty((T, 32, 128), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    dev.fill_kv(k, v, T, 0, 0, 1, stream=cs)
    out = {}
    for name, x in (("scatter", L), ("pack", 0)):
        assert kv.allocate_prefill(0, T, x)
        dev.set_timing(True)
        dev.offload_stats(reset=True)
        for layer in range(L):
            dev.prefill_layer(0, layer, k, v, T, stream=cs)
        dev.synchronize()
        st = dev.offload_stats(reset=True)
        ms = st.scatter_ms if name == "scatter" else st.pack_ms
        byts = 2 * T * 32 * 128 * 2 * 2 * L  # read K+V, write the slots
        out[name] = {"ms": ms, "hbm_gbs": byts / (ms / 1e3) / 1e9 if ms else None}
        if name == "scatter":  # escalation: gather every GPU slot of the request into staging + D2H
            job = kv.plan_offload(0, ls.FULL)
            dev.synchronize()
            kv.complete_offload(job.job_id)
        kv.release(0)
    print(json.dumps(out))
    dev.close()


if __name__ == "__main__":
    main()
