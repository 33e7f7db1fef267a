"""Parity of the sm_100a device path (calls go through the C ABI).

Bytes: bit-exact with the oracle generator (oracle/kvgen.c restated on the
device) after scatter, pack + D2H, escalation gather + D2H, and H2D prefetch.
Attention: fp32 output within 1e-3 relative (per row, max-abs normalised) of
the fp32 CPU restatement oracle/attn_ref.c; bf16 output within bf16 rounding.
"""
import numpy as np
import pytest

from paper_2410_00428_b200 import layersim as ls
from paper_2410_00428_b200.device import DTYPE_BF16, DTYPE_F32
from tests import _device_scenarios as sc

pytestmark = pytest.mark.gpu


def test_smoke_scenario():
    assert sc.smoke_scenario() <= sc.REL_TOL


@pytest.mark.parametrize("bs", [16, 32, 64])
@pytest.mark.parametrize("group", [1, 4])
def test_prefill_offload_bytes_bit_exact(bs, group):
    model = sc.gqa_model(L=6, hkv=4 if group == 4 else 8, group=group)
    kv, dev = sc.make(model, bs=bs, gpu=600, cpu=600, chunk_slots=2)
    prompts = [1, bs - 1, bs, bs + 1, 5 * bs + 3, 300]
    for rid, p in enumerate(prompts):
        sc.prefill(kv, dev, rid, p, rid % (model.n_layers + 1))
    for rid, p in enumerate(prompts):
        assert dev.verify_request(rid, p, sc.SEED) == 0
    # a wrong seed must be detected (the checker is not vacuous)
    assert dev.verify_request(4, prompts[4], sc.SEED + 1) > 0
    st = dev.offload_stats()
    assert st.d2h_bytes_algorithmic > 0 and st.scatter_bytes > 0


def test_host_frames_hold_slot_layout():
    """A pinned host frame holds exactly the oracle's slot bytes."""
    import oracle
    re = oracle.restatement()
    model = sc.gqa_model(L=2, hkv=8, group=1)
    kv, dev = sc.make(model)
    sc.prefill(kv, dev, 0, 40, 0)  # both layers on CPU
    r = kv.request(0)
    for b, blk in enumerate(r.blocks):
        for l, e in enumerate(blk.layers):
            assert e.loc == ls.LOC_CPU
            got = np.frombuffer(dev.read_host_slot(e.slot), np.uint16).reshape(2, 8, 16, 128)
            want = re.slot_bytes(l, b, 16, 8, 0, 128, 40, sc.SEED)
            assert np.array_equal(got, want)


@pytest.mark.parametrize("mode", [ls.HALF, ls.FULL])
def test_escalation_roundtrip(mode):
    model = sc.gqa_model(L=8, hkv=8, group=4)
    kv, dev = sc.make(model, gpu=800, cpu=800, chunk_slots=5)
    sc.prefill(kv, dev, 0, 170, 8)
    sc.prefill(kv, dev, 1, 90, 5)
    jobs = [kv.plan_offload(i, mode) for i in (0, 1)]
    for j in jobs:
        assert j.job_id >= 0
    for j in jobs:
        kv.complete_offload(j.job_id)
    kv.check_conservation()
    assert dev.verify_request(0, 170, sc.SEED) == 0
    assert dev.verify_request(1, 90, sc.SEED) == 0
    sc.check_attention(dev, [0, 1], [170, 90])


def test_release_during_inflight_escalation():
    model = sc.gqa_model(L=4, hkv=8, group=4)
    kv, dev = sc.make(model)
    sc.prefill(kv, dev, 0, 64, 4)
    job = kv.plan_offload(0, ls.FULL)
    f = kv.release(0)
    assert f.deferred_gpu == job.gpu_blocks
    kv.complete_offload(job.job_id)  # waits for the copy out of the send buffers
    kv.check_conservation()
    assert kv.gpu_blocks_free() == 512 and kv.cpu_blocks_free() == 512
    sc.prefill(kv, dev, 1, 64, 2)  # slots get reused
    assert dev.verify_request(1, 64, sc.SEED) == 0


@pytest.mark.parametrize("group,bs", [(1, 16), (2, 16), (4, 16), (8, 16), (4, 32), (1, 64), (8, 64)])
def test_attention_parity_ragged(group, bs):
    model = sc.gqa_model(L=3, hkv=8 if group < 8 else 4, group=group)
    kv, dev = sc.make(model, bs=bs, gpu=3000, cpu=3000, max_blocks=512, arena=3000)
    lens = [1, 7, bs, bs + 1, 333, 2500]
    for rid, n in enumerate(lens):
        sc.prefill(kv, dev, rid, n, rid % 4)
    sc.check_attention(dev, list(range(len(lens))), lens)


@pytest.mark.parametrize("group,bs", [(1, 16), (1, 32), (2, 32), (4, 16), (8, 16), (8, 64)])
def test_attention_parity_each_kernel(group, bs):
    """Both decode kernels (G = 1: persistent TMA-bulk CUDA-core kernel;
    G >= 2: tcgen05 GQA tile) against the fp32 oracle on ragged lengths,
    including chunks that end mid-tile and a sequence longer than one chunk."""
    model = sc.gqa_model(L=2, hkv=4, group=group)
    kv, dev = sc.make(model, bs=bs, gpu=4000, cpu=4000, max_blocks=640, arena=4000)
    lens = [1, 100, 129, 2 * bs + 3, 5000]
    for rid, n in enumerate(lens):
        sc.prefill(kv, dev, rid, n, rid % 3)
    sc.check_attention(dev, list(range(len(lens))), lens)


@pytest.mark.parametrize("group", [1, 8])
def test_attention_parity_merge_many_chunks(group):
    """The split merge (single pass, 4 warps, per-warp running max) on members
    with 1 to ~300 chunks, so batches cross the running-max rescale and warps
    see empty chunk lists."""
    model = sc.gqa_model(L=2, hkv=2, group=group)
    kv, dev = sc.make(model, gpu=9000, cpu=9000, max_blocks=4096, arena=9000)
    lens = [1, 40, 3000, 40000]
    for rid, n in enumerate(lens):
        sc.prefill(kv, dev, rid, n, rid % 3)
    sc.check_attention(dev, list(range(len(lens))), lens)


@pytest.mark.parametrize("mode", ["scaled", "rising", "extreme"])
@pytest.mark.parametrize("group,bs", [(1, 16), (2, 16), (4, 16), (8, 16), (4, 64)])
def test_attention_parity_peaked_softmax(mode, group, bs):
    """Peaked softmax (tests/_device_scenarios.peaked_q): scores whose running
    maximum rises tile after tile and chunk after chunk, so the tcgen05 tile's
    lazy max (decode_gqa_tc.cuh, raise when s > m_run + kLazyMax) fires mid
    sequence with its O/l correction, and the split merge rescales partials
    of different maxima. Lengths from 1 token to 40 chunks; some requests
    CPU-resident (arena frames)."""
    model = sc.gqa_model(L=2, hkv=4 if group < 8 else 2, group=group)
    kv, dev = sc.make(model, bs=bs, gpu=6000, cpu=6000, max_blocks=1400, arena=6000)
    lens = [1, 100, 129, 700, 5000, 20000]
    for rid, n in enumerate(lens):
        sc.prefill(kv, dev, rid, n, rid % 3)
    sc.check_attention(dev, list(range(len(lens))), lens, q_mode=mode)
    dev.close()


@pytest.mark.parametrize("mode", ["rising", "extreme"])
@pytest.mark.parametrize("group", [2, 4, 8])
def test_attention_parity_peaked_long_units(mode, group):
    """As above, with enough KV (8 KV heads x 4 x 40k tokens) that the tcgen05
    tile's chunking keeps 16-tile units (device.cu plan_chunks, the
    production shape: config 3's batch uses them too). Anchors then land deep
    inside a unit, so the in-tile lazy max raise and its O/l correction are
    what keeps the result right, not the split merge."""
    model = sc.gqa_model(L=2, hkv=8, group=group)
    lens = [40000, 39000, 40960, 37777]
    nb = sum((n + 15) // 16 for n in lens)
    kv, dev = sc.make(model, gpu=nb * 2 + 64, cpu=nb * 2 + 64, max_blocks=2600, arena=nb + 64, max_batch=4)
    for rid, n in enumerate(lens):
        sc.prefill(kv, dev, rid, n, 1 if rid % 2 else 0)
    sc.check_attention(dev, list(range(len(lens))), lens, layers=[1], q_mode=mode)
    dev.close()


@pytest.mark.parametrize("mode", [None, "rising"])
def test_attention_parity_bench_shape_g1(mode):
    """The headline's shape: LLaMA-2-7B heads (Hkv = Hq = 32, G = 1, the
    CUDA-core decode_attn_v2 kernel), 7 x 16384 tokens, every layer
    CPU-resident (x = 0, prefetched into the arena), all 32 heads of the last
    layer against the oracle."""
    model = ls.ModelSpec(2, 32, 32, 128, 4096, 7e9, 2)
    B, T, nblk = 7, 16384, 1024
    kv, dev = sc.make(model, gpu=64, cpu=B * nblk * 2 + 64, max_blocks=nblk + 8, max_batch=B,
                      arena=B * nblk + 16, chunk_slots=64)
    for rid in range(B):
        sc.prefill(kv, dev, rid, T, 0)
    sc.check_attention(dev, list(range(B)), [T] * B, layers=[1], q_mode=mode)
    dev.close()


@pytest.mark.parametrize("mode", [None, "rising"])
def test_attention_parity_70b_tp8_shard(mode):
    """Config 4's per-GPU shard at the a18 bench row's context: Llama-3.1-70B
    heads at TP 8, rank 7 (one KV head and its 8 query heads: G = 8 on the
    tcgen05 decode tile), 12 x 32768 tokens, layers GPU-resident, every query
    head of the last layer against the oracle (peaked softmax with "rising")."""
    model = ls.ModelSpec(2, 64, 8, 128, 8192, 70.6e9, 2)
    B, T, nblk = 12, 32768, 2048
    kv, dev = sc.make(model, gpu=B * nblk * 2 + 64, cpu=64, tp_rank=7, tp_size=8, max_blocks=nblk + 8,
                      max_batch=B, arena=B * nblk + 16)
    for rid in range(B):
        sc.prefill(kv, dev, rid, T, 2)
    sc.check_attention(dev, list(range(B)), [T] * B, layers=[1], q_mode=mode)
    dev.close()


def test_attention_bf16_output():
    model = sc.gqa_model(L=2, hkv=8, group=4)
    kv, dev = sc.make(model)
    sc.prefill(kv, dev, 0, 250, 1)
    sc.check_attention(dev, [0], [250], out_dtype=DTYPE_BF16)


def test_attention_long_context_splits():
    """Enough blocks that the split-K merge path runs with many splits."""
    model = sc.gqa_model(L=2, hkv=2, group=4)
    kv, dev = sc.make(model, gpu=9000, cpu=9000, max_blocks=4096, arena=9000)
    sc.prefill(kv, dev, 0, 40000, 1)
    sc.check_attention(dev, [0], [40000])


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_decode_after_appends_and_pipeline_depth(depth):
    """Decode blocks appended on CPU-resident layers are fetched too."""
    model = sc.gqa_model(L=5, hkv=8, group=4)
    kv, dev = sc.make(model, depth=depth)
    sc.prefill(kv, dev, 0, 30, 2)
    sc.prefill(kv, dev, 1, 16, 0)
    for rid in (0, 1):
        for _ in range(20):
            if kv.needs_append(rid):
                assert kv.append_decode_block(rid)
            kv.note_token(rid)
    for rid, n in ((0, 50), (1, 36)):
        dev.fill_request(rid, n, sc.SEED)  # decode-produced tokens (f2 write-back stand-in)
        assert dev.verify_request(rid, n, sc.SEED) == 0
    for _ in range(3):  # several iterations reuse the arena stages
        sc.check_attention(dev, [0, 1], [50, 36])


def test_kv_head_shards_compose():
    """TP=2: each shard owns half the KV heads; shard outputs concatenated over
    heads equal the single-GPU result (both checked against the oracle)."""
    model = sc.gqa_model(L=2, hkv=8, group=4)
    outs = []
    for r in range(2):
        kv, dev = sc.make(model, tp_rank=r, tp_size=2)
        sc.prefill(kv, dev, 0, 130, 1)
        assert dev.verify_request(0, 130, sc.SEED) == 0
        assert dev.q_heads_local == 16 and dev.head0 == 4 * r
        _, o = sc.check_attention(dev, [0], [130])
        outs.append(o)
        dev.close()
    assert outs[0][0].shape[1] + outs[1][0].shape[1] == model.n_heads


def test_decode_stats_accounting():
    model = sc.gqa_model(L=4, hkv=8, group=4)
    kv, dev = sc.make(model)
    sc.prefill(kv, dev, 0, 100, 2)
    dev.set_timing(True)
    sc.check_attention(dev, [0], [100])
    st = dev.decode_stats()
    kvb = 2 * 8 * 128 * 2
    fetch = sum(j.bytes for j in kv.plan_decode_fetch(0))
    assert st.h2d_bytes_algorithmic == fetch  # == reference plan_decode_fetch bytes
    assert st.kv_bytes_read == 100 * kvb * 4
    assert st.attn_launches == 4 and st.attn_ms > 0 and st.iteration_ms > 0
    # the kernels' own %globaltimer span sits inside the event-timed attention intervals
    assert 0 < st.kernel_ms <= st.attn_ms + 0.05


def test_capacity_error_is_loud():
    model = sc.gqa_model(L=2, hkv=8, group=4)
    kv, dev = sc.make(model, gpu=64, cpu=64)
    with pytest.raises(ls.CapacityError):
        dev.decode_begin(list(range(9)))  # > max_batch


def test_default_stream_inputs_are_ordered():
    """decode_layer with the caller on torch's default (legacy) stream: the
    caller's next write to q must wait until the attention read it (the
    regression: a NULL handle dropped the join, and a recycled q buffer was
    overwritten before layer 0's kernel ran)."""
    import math

    import numpy as np
    import torch
    import oracle
    from paper_2410_00428_b200.device import DTYPE_F32
    model = sc.gqa_model(L=1, hkv=8, group=1)
    kv, dev = sc.make(model, gpu=2000, cpu=2000, max_blocks=1300, arena=2000)
    n_tok = 20000  # offloaded: the attention waits for a 20k-token prefetch first
    sc.prefill(kv, dev, 0, n_tok, 0)
    q_host = sc.random_q(1, 8, 128, 99)
    q = q_host.to("cuda:0")
    out = torch.empty((1, 8, 128), dtype=torch.float32, device="cuda:0")
    dev.decode_begin([0])
    dev.decode_layer(0, q, out, 1 / math.sqrt(128), DTYPE_F32)  # stream=None: torch's current (default) stream
    q.fill_(7.0)  # default stream: must run after the kernel consumed q
    dev.decode_end()
    dev.synchronize()
    torch.cuda.synchronize()
    re = oracle.restatement()
    want = re.decode_attn_gen(sc.SEED, 0, n_tok, 0, 8, 1, q_host.view(torch.int16).numpy().view(np.uint16)[0],
                              1 / math.sqrt(128))
    got = out[0].cpu().numpy()
    err = np.abs(got - want).max(axis=-1) / np.abs(want).max(axis=-1)
    assert err.max() <= sc.REL_TOL


def test_table_journal_last_update_wins():
    """complete_offload, release and the next allocate_prefill can rewrite the
    same table entries before one flush; the device table must end with the
    last value (regression: the parallel apply raced on duplicate entries
    and a scatter went to a stale CPU-slot frame)."""
    model = sc.gqa_model(L=4, hkv=8, group=1)
    kv, dev = sc.make(model, gpu=3000, cpu=3000, max_blocks=200)
    for it in range(6):
        sc.prefill(kv, dev, 0, 1500, 4)  # every layer retained: scatter through the table row
        assert dev.verify_request(0, 1500, sc.SEED) == 0, f"iteration {it}"
        job = kv.plan_offload(0, ls.FULL)
        dev.synchronize()
        kv.complete_offload(job.job_id)  # journal: every entry -> its CPU slot
        kv.release(0)                    # the row returns to the free list, same row next time
    dev.close()


def test_free_list_mirror_after_rng31_fuzz():
    """a4: the device's HBM mirror of both LIFO free lists (table_apply_kernel
    applies the manager's free-list journal with the table journal) equals
    the host stacks after every op of the Rng(31) stream of
    test_kv_manager.cpp:265-322 — escalations, completions, orphaned
    releases included — and the host stacks equal the reference SlotPool's
    (tests/test_parity_bookkeeping.py::test_fuzz_free_stacks_vs_reference)."""
    from paper_2410_00428_b200.device import Device, DeviceConfig
    from tests import _drivers as drv
    model = ls.ModelSpec(8, 4, 4, 128, 512, 1e8, 2)  # the fuzz's 8 layers, d_head 128 for the device
    checked = []
    devs = []

    def bind(kv):
        dev = Device(kv, model, 16, DeviceConfig(device=0, gpu_slots=256, host_slots=512, arena_slots=64,
                                                 max_requests=160, max_blocks=40, max_batch=4, staging_chunks=4,
                                                 chunk_bytes=1 << 20))
        devs.append(dev)

        def check(step):
            if step % 7 and step != -1:
                return
            for gpu in (True, False):
                assert dev.free_stack(gpu) == kv.free_stack(gpu), (step, gpu)
            checked.append(step)
        return check
    drv.fuzz_ops(None, seed=31, rounds=3, steps=300, model=model, on_kv=bind)
    for d in devs:
        d.close()
    assert len(checked) > 100 and checked.count(-1) == 3


def test_offload_of_reused_slots_coalesces():
    """A released request's CPU slots come back off the LIFO free list in
    reverse order. The pack writes such a span into staging in reverse, so the
    D2H is still one copy per staging segment (round 2: every other prefill in
    the bench's a14 row issued one copy per block), and the bytes stay exact."""
    model = sc.gqa_model(L=2, hkv=8, group=1)
    kv, dev = sc.make(model, gpu=64, cpu=600, chunk_slots=64)
    prompt = 16 * 60  # 60 blocks per layer, one staging segment each
    copies = []
    for it in range(3):
        dev.offload_stats(reset=True)
        sc.prefill(kv, dev, it, prompt, 0)
        slots = [blk.layers[0].slot for blk in kv.request(it).blocks]
        assert slots == sorted(slots) or slots == sorted(slots, reverse=True)
        copies.append(dev.offload_stats().d2h_copies)
        assert dev.verify_request(it, prompt, sc.SEED) == 0
        kv.release(it)
    assert copies == [2, 2, 2], copies  # one copy per layer, ascending or descending slots
