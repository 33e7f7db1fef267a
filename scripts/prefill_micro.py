"""Prefill-attention microbenchmark (development aid): one causal GQA layer
through lkv_prefill_attention, CUDA-event timed on the launching stream.

  python scripts/prefill_micro.py [--tokens 32768] [--hq 32] [--hkv 8] [--iters 5]

FLOPs counted = 4 * d * Hq * T(T+1)/2 (QK^T + PV over the causal triangle),
the algorithmic count; the hi/lo split of P costs the tensor core one more PV.
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2410_00428_b200 import layersim as ls  # noqa: E402
from paper_2410_00428_b200.device import DTYPE_BF16, Device, DeviceConfig  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--tokens", type=int, default=32768)
    p.add_argument("--hq", type=int, default=32)
    p.add_argument("--hkv", type=int, default=8)
    p.add_argument("--iters", type=int, default=5)
    p.add_argument("--lib", default=None, help="an alternative liblkv.so (scripts/build_variant.sh)")
    p.add_argument("--label", default="product")
    a = p.parse_args()
    from paper_2410_00428_b200 import _abi
    lib = _abi.Lib(a.lib) if a.lib else None
    model = ls.ModelSpec(1, a.hq, a.hkv, 128, a.hq * 128, 8e9, 2)
    kv = ls.KvManager(ls.BlockPools(64, 64, 16), model, lib=lib)
    dev = Device(kv, model, 16, DeviceConfig(gpu_slots=64, host_slots=64, arena_slots=64, max_requests=2,
                                             max_blocks=64, max_batch=2), lib=lib)
    T = a.tokens
    q = (torch.rand((T, a.hq, 128), device="cuda") * 2 - 1).to(torch.bfloat16)
    k = (torch.rand((T, a.hkv, 128), device="cuda") * 2 - 1).to(torch.bfloat16)
    v = (torch.rand((T, a.hkv, 128), device="cuda") * 2 - 1).to(torch.bfloat16)
    out = torch.empty_like(q)
    s = dev.torch_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for it in range(a.iters + 2):
        torch.cuda.synchronize()
        e0.record(s)
        dev.prefill_attention(q, k, v, out, T, 1 / math.sqrt(128), DTYPE_BF16, stream=s)
        e1.record(s)
        e1.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
    ms = min(times)
    flops = 4.0 * 128 * a.hq * T * (T + 1) / 2
    peak = 1624.4  # round-1 figure, kept for comparability of the jsonl series
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            burst = json.load(f)["bf16_tflops"]
    except (OSError, KeyError, ValueError):
        burst = None
    print(json.dumps({"lib": a.label, "tokens": T, "hq": a.hq, "hkv": a.hkv, "ms": ms, "tflops": flops / ms / 1e9,
                      "frac_of_1624.4": flops / ms / 1e9 / peak,
                      "frac_of_measured_burst": flops / ms / 1e9 / burst if burst else None}))
    dev.close()


if __name__ == "__main__":
    main()
