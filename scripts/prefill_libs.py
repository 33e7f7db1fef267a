"""Library prefill attention on the same shapes as scripts/prefill_micro.py
(measurement aid, not product code): the best library kernel this image has
for causal GQA bf16 attention, timed the same way (CUDA events on the
launching stream, min of --iters after 2 warm-up launches), so the a20 row
can say how far the hand-written tcgen05 kernel is from it.

  python scripts/prefill_libs.py --backend cudnn|flashinfer-<b> [--tokens 16384]

cudnn: torch SDPA restricted to the cuDNN backend (K/V expanded to Hq heads
if the backend rejects GQA); flashinfer-<b>: flashinfer.single_prefill_with_kv_cache
with backend <b> (auto, cutlass, trtllm-gen, fa2, cudnn).
FLOPs counted as prefill_micro.py: 4 * d * Hq * T(T+1)/2.
"""
import argparse
import json
import math
import os
import sys

import torch


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--backend", required=True)
    p.add_argument("--tokens", type=int, default=16384)
    p.add_argument("--hq", type=int, default=32)
    p.add_argument("--hkv", type=int, default=8)
    p.add_argument("--iters", type=int, default=5)
    a = p.parse_args()
    T, d = a.tokens, 128
    torch.manual_seed(0)
    q = (torch.rand((T, a.hq, d), device="cuda") * 2 - 1).to(torch.bfloat16)
    k = (torch.rand((T, a.hkv, d), device="cuda") * 2 - 1).to(torch.bfloat16)
    v = (torch.rand((T, a.hkv, d), device="cuda") * 2 - 1).to(torch.bfloat16)
    scale = 1 / math.sqrt(d)
    note = None
    if a.backend == "cudnn":
        from torch.nn.attention import SDPBackend, sdpa_kernel
        qh = q.transpose(0, 1).unsqueeze(0)
        kh = k.transpose(0, 1).unsqueeze(0)
        vh = v.transpose(0, 1).unsqueeze(0)
        rep = a.hq // a.hkv
        kx = kh.repeat_interleave(rep, dim=1).contiguous()
        vx = vh.repeat_interleave(rep, dim=1).contiguous()
        qh = qh.contiguous()

        def run():
            with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
                return torch.nn.functional.scaled_dot_product_attention(qh, kx, vx, is_causal=True, scale=scale)
        note = "K/V expanded to Hq heads"
    elif a.backend.startswith("flashinfer-"):
        import flashinfer
        b = a.backend[len("flashinfer-"):]

        def run():
            return flashinfer.single_prefill_with_kv_cache(q, k, v, causal=True, sm_scale=scale, backend=b)
    else:
        raise SystemExit("unknown backend " + a.backend)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for it in range(a.iters + 2):
        torch.cuda.synchronize()
        e0.record(s)
        run()
        e1.record(s)
        e1.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
    ms = min(times)
    flops = 4.0 * d * a.hq * T * (T + 1) / 2
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
            burst = json.load(f)["bf16_tflops"]
    except (OSError, KeyError, ValueError):
        burst = None
    print(json.dumps({"lib": a.backend, "tokens": T, "hq": a.hq, "hkv": a.hkv, "ms": ms, "times_ms": times,
                      "tflops": flops / ms / 1e9, "frac_of_measured_burst": flops / ms / 1e9 / burst if burst else None,
                      "note": note}))


if __name__ == "__main__":
    sys.exit(main())
