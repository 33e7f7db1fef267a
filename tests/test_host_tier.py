"""Tiered host memory.

With pinned_frames > 0 every CPU slot lives in pageable memory and a small
pool of pinned frames carries the DMA traffic; a cleaner thread writes dirty
frames home and missing slots are read back on demand. The pinned pool here
is far smaller than the CPU slots in use, so every path (prefill pack + D2H,
escalation gather + D2H, per-layer prefetch, decode-time write-back, verify)
runs through evictions, write-backs and read-ins — and every byte must still
be bit-exact with the generator, every attention output within 1e-3."""
from __future__ import annotations

import pytest

from paper_2410_00428_b200 import layersim as ls
from tests import _device_scenarios as sc
from tests.test_decode_append import _decode_step

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("group,bs,pinned", [(1, 16, 40), (4, 16, 40), (8, 32, 44)])
def test_tiered_prefill_decode_append_bit_exact(group, bs, pinned):
    model = sc.gqa_model(L=4, hkv=2, group=group)
    kv, dev = sc.make(model, bs=bs, gpu=600, cpu=600, max_blocks=64, arena=300, pinned=pinned)
    prompts = {0: 5 * bs + 3, 1: 3 * bs, 2: 7 * bs + 5}
    xs = {0: 0, 1: 2, 2: 1}
    for rid, p in prompts.items():
        sc.prefill(kv, dev, rid, p, xs[rid])
    ids = list(prompts)
    cpu_slots = 600 - kv.cpu_blocks_free()
    assert cpu_slots > pinned  # the working set does not fit the pinned frames
    sc.check_attention(dev, ids, [prompts[r] for r in ids])
    for _ in range(bs + 3):
        _decode_step(kv, dev, ids)
    kv.check_conservation()
    for rid in ids:
        n = kv.request(rid).cached_tokens
        assert dev.verify_request(rid, n, sc.SEED) == 0, f"request {rid}"
    st = dev.host_tier_stats()
    assert st.pinned_frames == pinned
    assert st.evictions > 0 and st.read_in_frames > 0 and st.write_back_frames > 0
    dev.close()


def test_tiered_escalation_and_release_reuse():
    """An escalation's D2H lands in pinned frames and is written home; after
    release the freed slots are reused by a new request whose bytes must not
    be confused with the old ones."""
    model = sc.gqa_model(L=4, hkv=2, group=4)
    kv, dev = sc.make(model, bs=16, gpu=600, cpu=600, max_blocks=64, arena=300, pinned=32)
    sc.prefill(kv, dev, 0, 90, 4)
    sc.prefill(kv, dev, 1, 70, 0)
    job = kv.plan_offload(0, ls.FULL)
    assert job is not None and job.job_id >= 0
    _decode_step(kv, dev, [0, 1])
    kv.complete_offload(job.job_id)
    for _ in range(5):
        _decode_step(kv, dev, [0, 1])
    for rid in (0, 1):
        assert dev.verify_request(rid, kv.request(rid).cached_tokens, sc.SEED) == 0
    kv.release(1)
    sc.prefill(kv, dev, 2, 100, 0, seed=sc.SEED)  # reuses request 1's CPU slots (LIFO)
    for _ in range(4):
        _decode_step(kv, dev, [0, 2])
    for rid in (0, 2):
        assert dev.verify_request(rid, kv.request(rid).cached_tokens, sc.SEED) == 0
    # a host slot read through the C ABI equals the generator restatement
    import numpy as np
    import oracle
    re = oracle.restatement()
    r2 = kv.request(2)
    for b in (0, 3):
        e = r2.blocks[b].layers[0]
        assert e.loc == ls.LOC_CPU
        got = np.frombuffer(dev.read_host_slot(e.slot), np.uint16).reshape(2, dev.kv_heads_local, 16, 128)
        want = re.slot_bytes(0, b, 16, dev.kv_heads_local, dev.head0, 128, r2.cached_tokens, sc.SEED)
        assert np.array_equal(got, want)
    dev.close()


def test_tiered_pinned_pool_too_small_is_loud():
    model = sc.gqa_model(L=2, hkv=2, group=1)
    kv, dev = sc.make(model, bs=16, gpu=64, cpu=600, max_blocks=64, arena=300, pinned=4)
    with pytest.raises(ls.CapacityError):
        sc.prefill(kv, dev, 0, 16 * 40, 0)
        sc.check_attention(dev, [0], [16 * 40])  # one layer's prefetch needs 40 frames at once
    dev.close()

