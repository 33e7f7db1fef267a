"""Stress the ragged decode-attention scenario (development aid): repeats
tests/test_device_gpu.py::test_attention_parity_ragged and reports, on any
mismatch, which request/layer failed and whether the KV bytes themselves
(verify_request) are intact.

  python scripts/stress_ragged.py [--iters 20] [--group 1] [--bs 16] [--kernel 2]
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2410_00428_b200.device import DTYPE_F32  # noqa: E402
from tests import _device_scenarios as sc  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--iters", type=int, default=20)
    p.add_argument("--group", type=int, default=1)
    p.add_argument("--bs", type=int, default=16)
    a = p.parse_args()
    re = oracle.restatement()
    fails = 0
    for it in range(a.iters):
        model = sc.gqa_model(L=3, hkv=8 if a.group < 8 else 4, group=a.group)
        kv, dev = sc.make(model, bs=a.bs, gpu=3000, cpu=3000, max_blocks=512, arena=3000)
        lens = [1, 7, a.bs, a.bs + 1, 333, 2500]
        for rid, n in enumerate(lens):
            sc.prefill(kv, dev, rid, n, rid % 4)
        bad_bytes = [dev.verify_request(rid, n, sc.SEED) for rid, n in enumerate(lens)]
        n = len(lens)
        hq, d = dev.q_heads_local, dev.head_dim
        qs = [sc.random_q(n, hq, d, 1000 + l) for l in range(3)]
        outs = []
        dev.decode_begin(list(range(n)))
        for l in range(3):
            out = torch.empty((n, hq, d), dtype=torch.float32, device="cuda:0")
            dev.decode_layer(l, qs[l].cuda(), out, 1 / math.sqrt(d), DTYPE_F32)
            outs.append(out)
        dev.decode_end()
        dev.synchronize()
        msgs = []
        for l in range(3):
            got = outs[l].cpu().numpy()
            q16 = qs[l].view(torch.int16).numpy().view(np.uint16)
            for m in range(n):
                want = re.decode_attn_gen(sc.SEED, l, lens[m], 0, dev.kv_heads_local, hq // dev.kv_heads_local,
                                          q16[m], 1 / math.sqrt(d))
                err = np.abs(got[m] - want).max(axis=-1) / np.maximum(np.abs(want).max(axis=-1), 1e-30)
                if err.max() > 1e-3:
                    heads = np.nonzero(err > 1e-3)[0]
                    msgs.append(f"layer {l} member {m} (len {lens[m]}, x {m % 4}) heads {heads.tolist()[:8]} "
                                f"err {err.max():.3e} got[0,:4] {got[m, heads[0], :4]} want {want[heads[0], :4]}")
        if msgs or any(bad_bytes):
            fails += 1
            print(f"iter {it}: bytes mismatches {bad_bytes}")
            for s in msgs[:12]:
                print("   ", s)
        dev.close()
        del kv
    print(f"{fails} / {a.iters} iterations failed")


if __name__ == "__main__":
    main()
