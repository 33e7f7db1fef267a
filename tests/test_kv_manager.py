"""Restatement of proj/tests/test_kv_manager.cpp (every TEST_CASE), run against
the product library and, where present, against the compiled reference — the
same assertions must hold for both."""
import pytest

from paper_2410_00428_b200 import layersim as ls
from paper_2410_00428_b200.layersim import FULL, HALF, LOC_CPU, LOC_GPU


@pytest.fixture(params=["product", "reference"])
def lib(request, prod):
    if request.param == "product":
        return prod
    return request.getfixturevalue("ref")


def l20():
    return ls.HardwareSpec(1.0e14, 8.64e11, 3.2e10, False, 1, 48e9, 0.9)


def small(lib, gpu, cpu, m):
    return ls.KvManager(ls.BlockPools(gpu, cpu, 16), m, lib=lib)


def test_pool_sizing_formula(lib):  # test_kv_manager.cpp:33-54
    s = ls.PoolSizing(16384, 16, 4.0, 8.0)
    p = ls.pool_size_from_hardware(ls.llama2_7b(), l20(), s, lib=lib)
    assert p.gpu_blocks_total == 113043
    assert p.cpu_blocks_total == 113043 * 8
    p2 = ls.pool_size_from_hardware(ls.llama2_7b(), l20(), ls.PoolSizing(32768, 16, 4.0, 8.0), lib=lib)
    assert p2.gpu_blocks_total < p.gpu_blocks_total
    hw = l20()
    hw.gpu_mem = 10e9
    with pytest.raises(ls.ConfigError):
        ls.pool_size_from_hardware(ls.llama2_7b(), hw, s, lib=lib)


def test_pool_sizing_b200_configs(lib):  # B200 180 GB / 8B / 32k and 70B TP8
    hw = ls.HardwareSpec(1.3814e15, 6.5367e12, 5.5e10, True, 1, 180e9, 0.9)
    p = ls.pool_size_from_hardware(ls.llama3_8b_gqa(), hw, ls.PoolSizing(32768, 16, 4.0, 8.0), lib=lib)
    assert p.gpu_blocks_total == 2221882
    hw.n_gpus = 8
    p = ls.pool_size_from_hardware(ls.llama31_70b_gqa(), hw, ls.PoolSizing(16384, 16, 4.0, 8.0), lib=lib)
    assert p.gpu_blocks_total > 0


def test_layer_placement_examples(lib):  # :56-64
    p = ls.layer_placement(8, 4, lib=lib)
    assert p.retained == [1, 3, 5, 7] and p.offloaded == [0, 2, 4, 6]
    assert ls.layer_placement(8, 0, lib=lib).retained == []
    assert len(ls.layer_placement(8, 0, lib=lib).offloaded) == 8
    assert ls.layer_placement(8, 3, lib=lib).retained == [1, 4, 6]
    with pytest.raises(ls.DomainError):
        ls.layer_placement(8, 9, lib=lib)


@pytest.mark.parametrize("L", [1, 2, 8, 32, 60, 80, 127])
def test_layer_placement_distinct(lib, L):  # :66-80
    for x in range(L + 1):
        p = ls.layer_placement(L, x, lib=lib)
        assert len(set(p.retained)) == x
        assert all(0 <= l < L for l in p.retained)
        assert len(p.retained) + len(p.offloaded) == L


def test_allocate_prefill_splits(lib):  # :82-102
    m = ls.llama2_7b()
    kv = small(lib, 10000, 10000, m)
    assert kv.allocate_prefill(1, 2048, 0)
    assert kv.gpu_blocks_free() == 10000 and kv.cpu_blocks_free() == 10000 - 32 * 128
    kv = small(lib, 10000, 10000, m)
    need = kv.request_wise_gpu_blocks(2048)
    assert kv.allocate_prefill(1, 2048, 32)
    assert kv.gpu_blocks_free() == 10000 - need and kv.cpu_blocks_free() == 10000
    kv = small(lib, 10000, 10000, m)
    assert kv.allocate_prefill(1, 2048, 8)
    assert kv.gpu_blocks_free() == 10000 - 8 * 128 and kv.cpu_blocks_free() == 10000 - 24 * 128


def test_allocation_failure_atomic(lib):  # :104-113
    kv = small(lib, 100, 50, ls.llama2_7b())
    assert not kv.allocate_prefill(1, 2048, 8)
    assert kv.gpu_blocks_free() == 100 and kv.cpu_blocks_free() == 50
    assert not kv.has_request(1)
    kv.check_conservation()


def test_no_shared_slots(lib):  # :115-132
    kv = small(lib, 64, 64, ls.tiny8())
    assert kv.allocate_prefill(1, 16, 4) and kv.allocate_prefill(2, 16, 4)
    kv.check_conservation()
    seen = set()
    for rid in (1, 2):
        for blk in kv.request(rid).blocks:
            for e in blk.layers:
                if e.loc == LOC_GPU:
                    assert e.slot not in seen
                    seen.add(e.slot)
    assert len(seen) == 8


def test_plan_offload_half_then_full(lib):  # :134-159
    m = ls.tiny8()
    kv = small(lib, 64, 64, m)
    assert kv.allocate_prefill(1, 16, 4)
    assert kv.retained_layer_count(1) == 4
    half = kv.plan_offload(1, HALF)
    assert half.layer_count == 2 and half.gpu_blocks == 2
    assert half.bytes == 2.0 * 16 * ls.kv_bytes_per_token_layer(m, lib=lib)
    kv.complete_offload(half.job_id)
    assert kv.retained_layer_count(1) == 2
    full = kv.plan_offload(1, FULL)
    assert full.layer_count == 2
    kv.complete_offload(full.job_id)
    assert kv.retained_layer_count(1) == 0 and kv.gpu_blocks_free() == 64
    nothing = kv.plan_offload(1, HALF)
    assert nothing.job_id == -1 and nothing.layer_count == 0


def test_send_buffers_held_until_complete(lib):  # :161-172
    kv = small(lib, 64, 64, ls.tiny8())
    assert kv.allocate_prefill(1, 16, 8)
    before = kv.gpu_blocks_free()
    job = kv.plan_offload(1, HALF)
    assert kv.gpu_blocks_free() == before
    kv.check_conservation()
    kv.complete_offload(job.job_id)
    assert kv.gpu_blocks_free() == before + job.gpu_blocks


def test_plan_decode_fetch(lib):  # :174-193
    m = ls.llama2_7b()
    kv = small(lib, 100000, 100000, m)
    assert kv.allocate_prefill(1, 2048, 32)
    assert kv.plan_decode_fetch(1) == []
    kv = small(lib, 100000, 100000, m)
    assert kv.allocate_prefill(1, 2048, 16)
    jobs = kv.plan_decode_fetch(1)
    assert len(jobs) == 16
    assert [j.layer for j in jobs] == sorted(j.layer for j in jobs)
    assert all(j.bytes == 2048.0 * 16384.0 for j in jobs)


def test_append_follows_residency(lib):  # :195-229
    m = ls.tiny8()
    kv = small(lib, 64, 64, m)
    assert kv.allocate_prefill(1, 10, 8)
    assert not kv.needs_append(1)
    kv.note_token(1)
    assert not kv.needs_append(1)
    kv = small(lib, 64, 64, m)
    assert kv.allocate_prefill(1, 16, 0) and kv.needs_append(1)
    g, c = kv.gpu_blocks_free(), kv.cpu_blocks_free()
    assert kv.append_decode_block(1)
    assert kv.gpu_blocks_free() == g and kv.cpu_blocks_free() == c - 8
    kv = small(lib, 64, 64, m)
    assert kv.allocate_prefill(1, 16, 8)
    g = kv.gpu_blocks_free()
    assert kv.append_decode_block(1)
    assert kv.gpu_blocks_free() == g - 8
    tight = small(lib, 8, 4, m)
    assert tight.allocate_prefill(2, 16, 8) and tight.needs_append(2)
    assert not tight.append_decode_block(2)
    assert tight.gpu_blocks_free() == 0 and tight.cpu_blocks_free() == 4


def test_release_and_double_release(lib):  # :231-244
    kv = small(lib, 64, 64, ls.tiny8())
    assert kv.allocate_prefill(1, 30, 4)
    while not kv.needs_append(1) and kv.request(1).cached_tokens < 32:
        kv.note_token(1)
    if kv.needs_append(1):
        kv.append_decode_block(1)
    f = kv.release(1)
    assert kv.gpu_blocks_free() == 64 and kv.cpu_blocks_free() == 64
    assert f.gpu + f.cpu > 0
    with pytest.raises(ls.SimulationError):
        kv.release(1)
    with pytest.raises(ls.SimulationError):
        kv.release(999)


def test_release_during_inflight_offload(lib):  # :246-263
    kv = small(lib, 64, 64, ls.tiny8())
    assert kv.allocate_prefill(1, 16, 8)
    job = kv.plan_offload(1, FULL)
    assert job.gpu_blocks == 8
    f = kv.release(1)
    assert f.deferred_gpu == 8 and kv.gpu_blocks_free() == 56
    kv.check_conservation()
    kv.complete_offload(job.job_id)
    assert kv.gpu_blocks_free() == 64 and kv.cpu_blocks_free() == 64
    kv.check_conservation()


def test_dump_format(lib):  # :324-333
    kv = small(lib, 64, 64, ls.tiny8())
    assert kv.allocate_prefill(7, 16, 4)
    d = kv.dump_table()
    assert "req=7 block=0 layer=0 -> CPU(" in d
    assert "req=7 block=0 layer=1 -> GPU(" in d


def test_error_conventions(lib):
    kv = small(lib, 64, 64, ls.tiny8())
    with pytest.raises(ls.SimulationError):
        kv.request(5)
    with pytest.raises(ls.SimulationError):
        kv.complete_offload(123)
    assert kv.allocate_prefill(1, 16, 8)
    with pytest.raises(ls.SimulationError):
        kv.allocate_prefill(1, 16, 8)
    with pytest.raises(ls.SimulationError):
        kv.note_token(1)  # block full: token past capacity
    with pytest.raises(ls.DomainError):
        kv.allocate_prefill(2, 16, 9)


def test_rollback_permutes_cpu_stack(lib):
    """a failed plan_offload pushes reserved CPU slots back in
    reservation order, so the next pops come out reversed (5, 4 not 4, 5)."""
    m = ls.ModelSpec(1, 4, 4, 32, 128, 1e8, 2)
    kv = small(lib, 64, 6, m)
    # 4 CPU slots used by an x=0 request of 64 tokens (4 blocks, 1 layer)
    assert kv.allocate_prefill(1, 64, 0)
    # a GPU-resident request with 3 blocks cannot find 3 CPU destinations (2 left)
    assert kv.allocate_prefill(2, 48, 1)
    assert kv.plan_offload(2, FULL) is None
    assert kv.allocate_prefill(3, 32, 0)
    slots = [blk.layers[0].slot for blk in kv.request(3).blocks]
    assert slots == [5, 4]
    kv.check_conservation()


def test_stale_dest_slot_after_rollback_is_visible(lib):
    """The reference leaves dest_slot set after a rollback (kv_manager.cpp:244-248)."""
    m = ls.ModelSpec(1, 4, 4, 32, 128, 1e8, 2)
    kv = small(lib, 64, 1, m)
    assert kv.allocate_prefill(2, 48, 1)
    assert kv.plan_offload(2, FULL) is None
    ents = [blk.layers[0] for blk in kv.request(2).blocks]
    assert ents[0].dest_slot == 0 and not ents[0].offload_in_flight
    assert all(e.loc == LOC_GPU for e in ents)
    assert kv.cpu_blocks_free() == 1


def test_counters_match_full_scans(lib):
    """O(L) counters (product) must equal the reference's O(blocks x L) scans."""
    m = ls.tiny8()
    kv = small(lib, 200, 200, m)
    assert kv.allocate_prefill(1, 40, 5)
    for _ in range(30):
        if kv.needs_append(1):
            assert kv.append_decode_block(1)
        kv.note_token(1)
    j = kv.plan_offload(1, HALF)
    r = kv.request(1)
    held = sum(e.loc == LOC_GPU for b in r.blocks for e in b.layers)
    assert kv.gpu_blocks_held(1) == held
    live_layers = {l for b in r.blocks for l, e in enumerate(b.layers) if e.loc == LOC_GPU and not e.offload_in_flight}
    assert kv.retained_layer_count(1) == len(live_layers)
    kv.complete_offload(j.job_id)
    r = kv.request(1)
    for job in kv.plan_decode_fetch(1):
        toks = sum(min(max(r.cached_tokens - b.token_begin, 0), 16) for b in r.blocks
                   if b.layers[job.layer].loc == LOC_CPU)
        assert job.bytes == toks * ls.kv_bytes_per_token_layer(m, lib=lib)


def test_free_delta_journal_replays_the_stacks():
    """a4: the free-list journal the device mirror applies (lkv_kv_free_delta)
    rebuilds both LIFO stacks exactly when replayed into a host-side mirror
    after every op of the Rng(31) fuzz (escalations, completions, orphaned
    releases) — including steps whose only change is a pop from the pushed
    part (the stack shrinks with nothing to upload: the header must still
    change; round 1's journal missed exactly that)."""
    from tests import _drivers as drv
    mirrors = []

    def bind(kv):
        total = {True: kv.gpu_blocks_total(), False: kv.cpu_blocks_total()}
        state = {g: {"fresh": 0, "pushed": []} for g in (True, False)}
        first = [True]

        def check(step):
            for g in (True, False):
                nf, lo, sz, changed, entries = kv.free_delta(g, full=first[0])
                st = state[g]
                if changed:
                    st["fresh"] = nf
                    st["pushed"] = st["pushed"][:lo] + entries
                    assert len(st["pushed"]) == sz
                mirror = list(range(total[g] - 1, st["fresh"] - 1, -1)) + st["pushed"]
                assert mirror == kv.free_stack(g), (step, g)
            first[0] = False
            mirrors.append(step)
        return check
    drv.fuzz_ops(None, seed=31, rounds=3, steps=300, on_kv=bind)
    assert len(mirrors) == 3 * 301


def test_rel_err_rows_counts_nan_as_failure():
    """The attention parity checks' error metric: a NaN or inf output row is
    an infinite error (max() and > both ignore NaN otherwise)."""
    import numpy as np
    from tests import _device_scenarios as sc
    want = np.ones((3, 4), np.float32)
    got = want.copy()
    assert sc.rel_err_rows(got, want).max() == 0.0
    got[1, 2] = np.nan
    assert np.isinf(sc.rel_err_rows(got, want)[1])
    got[1, 2] = np.inf
    assert np.isinf(sc.rel_err_rows(got, want).max())
