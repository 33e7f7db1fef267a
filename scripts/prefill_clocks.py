"""Clocks and power while the prefill attention runs back to back (development
aid): is the tensor-core kernel held by the power cap?

  python scripts/prefill_clocks.py [--lib ...] [--tokens 32768] [--seconds 4]
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

import bench  # noqa: E402
from paper_2410_00428_b200 import _abi  # noqa: E402
from paper_2410_00428_b200 import layersim as ls  # noqa: E402
from paper_2410_00428_b200.device import DTYPE_BF16, Device, DeviceConfig  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--lib", default=None)
    p.add_argument("--label", default="product")
    p.add_argument("--tokens", type=int, default=32768)
    p.add_argument("--seconds", type=float, default=4.0)
    p.add_argument("--cudnn", action="store_true", help="time torch SDPA (cuDNN backend, K/V expanded) instead")
    a = p.parse_args()
    lib = _abi.Lib(a.lib) if a.lib else None
    model = ls.ModelSpec(1, 32, 8, 128, 4096, 8e9, 2)
    kv = ls.KvManager(ls.BlockPools(64, 64, 16), model, lib=lib)
    dev = Device(kv, model, 16, DeviceConfig(gpu_slots=64, host_slots=64, arena_slots=64, max_requests=2,
                                             max_blocks=64, max_batch=2), lib=lib)
    T = a.tokens
    q = (torch.rand((T, 32, 128), device="cuda") * 2 - 1).to(torch.bfloat16)
    k = (torch.rand((T, 8, 128), device="cuda") * 2 - 1).to(torch.bfloat16)
    v = (torch.rand((T, 8, 128), device="cuda") * 2 - 1).to(torch.bfloat16)
    out = torch.empty_like(q)
    run = lambda: dev.prefill_attention(q, k, v, out, T, 1 / math.sqrt(128), DTYPE_BF16)  # noqa: E731
    if a.cudnn:  # the library kernel on the same shape, for the sustained comparison only
        from torch.nn.attention import SDPBackend, sdpa_kernel
        qh = q.transpose(0, 1).unsqueeze(0).contiguous()
        kx = k.transpose(0, 1).unsqueeze(0).repeat_interleave(4, dim=1).contiguous()
        vx = v.transpose(0, 1).unsqueeze(0).repeat_interleave(4, dim=1).contiguous()

        def run():
            with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
                torch.nn.functional.scaled_dot_product_attention(qh, kx, vx, is_causal=True, scale=1 / math.sqrt(128))
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    with bench.ClockSampler(0) as clk:
        t0 = time.perf_counter()
        e0.record()
        while time.perf_counter() - t0 < a.seconds:
            for _ in range(8):
                run()
                n += 1
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    flops = 4.0 * 128 * 32 * T * (T + 1) / 2
    power = [float(r[3]) for r in clk.rows if len(r) > 3 and r[3].replace(".", "").isdigit()]
    print(json.dumps({"lib": a.label, "tokens": T, "launches": n, "ms": ms, "tflops": flops / ms / 1e9,
                      "clocks": clk.summary(), "power_w_median": sorted(power)[len(power) // 2] if power else None}))
    dev.close()


if __name__ == "__main__":
    main()
