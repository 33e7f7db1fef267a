"""Decode-time KV write-back.

The reference allocates a slot for every decoded token (append_decode_block,
kv_manager.cpp:313-334; note_token 336-344) but never schedules its bytes.
The device path writes each new token's K/V wherever its slot lives (GPU
slot; CPU slot's pinned frame + this step's arena copy; both ends of an
in-flight offload) and attends over cached_tokens + 1 keys. Checked against
the oracle: every KV element of every layer bit-exact with the generator
after many steps (crossing block boundaries, escalations in flight), and
every step's attention within 1e-3 of the fp32 restatement.
"""
import math

import numpy as np
import pytest

from paper_2410_00428_b200 import layersim as ls
from tests import _device_scenarios as sc

pytestmark = pytest.mark.gpu


def _new_token_kv(dev, ids, kv, layer):
    """Generator K/V of each member's next token (position cached_tokens)."""
    import torch
    n = len(ids)
    k = torch.empty((n, dev.kv_heads_local, dev.head_dim), dtype=torch.bfloat16, device="cuda:0")
    v = torch.empty_like(k)
    s = dev.torch_stream("compute")
    for m, rid in enumerate(ids):
        dev.fill_kv(k[m], v[m], 1, kv.request(rid).cached_tokens, layer, sc.SEED, stream=s)
    return k, v


def _decode_step(kv, dev, ids, check=True):
    import torch
    import oracle
    from paper_2410_00428_b200.device import DTYPE_F32
    for rid in ids:  # engine.cpp:408-409
        if kv.needs_append(rid):
            assert kv.append_decode_block(rid)
    lens = [kv.request(rid).cached_tokens + 1 for rid in ids]
    L, hq, d = dev.model.n_layers, dev.q_heads_local, dev.head_dim
    qs = [sc.random_q(len(ids), hq, d, 77 + l + 10 * lens[0]) for l in range(L)]
    outs = []
    dev.decode_begin_append(ids)
    for l in range(L):
        k, v = _new_token_kv(dev, ids, kv, l)
        dev.decode_append_layer(l, k, v)
        out = torch.empty((len(ids), hq, d), dtype=torch.float32, device="cuda:0")
        dev.decode_layer(l, qs[l].cuda(), out, 1 / math.sqrt(d), DTYPE_F32)
        outs.append((out, k, v))
    dev.decode_end()
    dev.synchronize()
    worst = 0.0
    if check:
        re = oracle.restatement()
        group = hq // dev.kv_heads_local
        for l in range(L):
            got = outs[l][0].cpu().numpy()
            q16 = qs[l].view(torch.int16).numpy().view(np.uint16)
            for m in range(len(ids)):
                want = re.decode_attn_gen(sc.SEED, l, lens[m], dev.head0, dev.kv_heads_local, group, q16[m],
                                          1 / math.sqrt(d))
                worst = max(worst, float(sc.rel_err_rows(got[m], want).max()))
        assert worst <= sc.REL_TOL, f"attention rel err {worst:.3e}"
    for rid in ids:  # engine.cpp:151
        kv.note_token(rid)
    return worst


@pytest.mark.parametrize("group,bs", [(1, 16), (4, 16), (8, 32)])
def test_append_steps_bit_exact(group, bs):
    model = sc.gqa_model(L=4, hkv=2, group=group)
    kv, dev = sc.make(model, bs=bs, gpu=600, cpu=600, max_blocks=64, arena=300)
    prompts = {0: bs - 3, 1: bs, 2: 2 * bs + 5}   # mid-block, exactly full, multi-block
    xs = {0: 2, 1: 0, 2: 4}                        # half, none, all layers retained
    for rid, p in prompts.items():
        sc.prefill(kv, dev, rid, p, xs[rid])
    ids = list(prompts)
    for _ in range(bs + 4):  # crosses a block boundary for every member
        _decode_step(kv, dev, ids)
    kv.check_conservation()
    for rid in ids:
        n = kv.request(rid).cached_tokens
        assert n == prompts[rid] + bs + 4
        assert dev.verify_request(rid, n, sc.SEED) == 0, f"request {rid}"
    dev.close()


def test_append_during_inflight_escalation_and_after():
    """plan_offload flips layer_residency at once (kv_manager.cpp:236): the
    steps between plan and complete write the GPU slot and the destination
    frame; after completion new blocks of offloaded layers come from the CPU
    pool (N6)."""
    model = sc.gqa_model(L=4, hkv=2, group=4)
    kv, dev = sc.make(model, bs=16, gpu=600, cpu=600, max_blocks=64, arena=300)
    sc.prefill(kv, dev, 0, 30, 4)
    sc.prefill(kv, dev, 1, 40, 2)
    ids = [0, 1]
    _decode_step(kv, dev, ids)
    job = kv.plan_offload(0, ls.HALF)
    assert job is not None and job.job_id >= 0
    for _ in range(3):  # offload in flight: entries still GPU with a dest frame
        _decode_step(kv, dev, ids)
    kv.complete_offload(job.job_id)
    for _ in range(20):
        _decode_step(kv, dev, ids)
    kv.check_conservation()
    for rid in ids:
        n = kv.request(rid).cached_tokens
        assert dev.verify_request(rid, n, sc.SEED) == 0, f"request {rid}"
    dev.close()


def test_append_requires_block_and_order():
    from paper_2410_00428_b200 import _abi
    model = sc.gqa_model(L=2, hkv=2, group=1)
    kv, dev = sc.make(model, bs=16)
    sc.prefill(kv, dev, 0, 16, 1)
    # a full last block and no append_decode_block: there is no slot for the token
    with pytest.raises(_abi.LkvError):
        dev.decode_begin_append([0])
    assert kv.append_decode_block(0)
    dev.decode_begin_append([0])
    import torch
    q = torch.zeros((1, dev.q_heads_local, 128), dtype=torch.bfloat16, device="cuda:0")
    out = torch.empty_like(q)
    with pytest.raises(_abi.LkvError):  # decode_layer before the layer's append
        dev.decode_layer(0, q, out, 0.1)
    dev.decode_end()
    dev.close()
