"""Bit-exact parity of the product bookkeeping with the reference.

* committed golden fixtures (generated from the compiled reference by
  tests/golden/make_golden.py) — these run everywhere, also on the GPU box;
* live call-by-call comparison with the compiled reference (here).
"""
import random

import pytest

from paper_2410_00428_b200 import layersim as ls
from tests import _drivers as drv


# ---------------------------------------------------------------- goldens
@pytest.mark.parametrize("x", [0, 16, 32])
def test_config1_table_goldens(prod, golden, x):
    """FNV-1a of dump_table after prefill and after 64 tokens."""
    g = golden["kv"][f"cfg1_x{x}"]
    kv = ls.KvManager(ls.BlockPools(200000, 800000, 16), ls.llama2_7b(), lib=prod)
    assert kv.allocate_prefill(0, 1024, x)
    assert format(kv.dump_hash(), "016x") == g["after_prefill"]
    for _ in range(64):
        if kv.needs_append(0):
            assert kv.append_decode_block(0)
        kv.note_token(0)
    assert format(kv.dump_hash(), "016x") == g["after_64"]
    assert (kv.gpu_blocks_free(), kv.cpu_blocks_free()) == (g["gpu_free"], g["cpu_free"])
    assert [[j.layer, j.bytes] for j in kv.plan_decode_fetch(0)] == g["fetch"]


def test_baseline_md_hashes_literal(prod):
    """The hashes printed in BASELINE.md §2 themselves."""
    want = {0: ("df568e8882f46775", "b711b4e97b65e8af"), 16: ("3e60c733e013b905", "bee031c29dee178b"),
            32: ("131d145cdb9b3ea5", "30fb82b667d28c2f")}
    for x, (a, b) in want.items():
        kv = ls.KvManager(ls.BlockPools(200000, 800000, 16), ls.llama2_7b(), lib=prod)
        kv.allocate_prefill(0, 1024, x)
        assert format(kv.dump_hash(), "016x") == a
        for _ in range(64):
            if kv.needs_append(0):
                kv.append_decode_block(0)
            kv.note_token(0)
        assert format(kv.dump_hash(), "016x") == b


def test_fuzz_rng31_matches_golden(prod, golden):
    """proj/tests/test_kv_manager.cpp:265-322 op stream (Rng 31, 10 x 300):
    every return value, free count and table hash after every op."""
    trace = drv.fuzz_ops(prod)
    g = golden["kv"]["fuzz_rng31"]
    assert drv.trace_digest(trace) == g["digest"], _first_diff(trace[0], g["round0"])


def test_fuzz_tight_pools_matches_golden(prod, golden):
    """Tight pools: many rolled-back plan_offloads and failed appends."""
    trace = drv.fuzz_ops(prod, seed=2024, rounds=6, steps=400, gpu=96, cpu=64, max_prompt=48)
    g = golden["kv"]["fuzz_tight_2024"]
    assert drv.trace_digest(trace) == g["digest"], _first_diff(trace[0], g["round0"])


def _first_diff(a, b):
    import json
    a = json.loads(json.dumps(a))
    for i, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return f"first difference at op {i}: product {x} vs reference {y}"
    return "traces differ in later rounds"


# ---------------------------------------------------------------- live vs reference
@pytest.mark.parametrize("seed", [1, 7, 99, 31337])
def test_fuzz_live_vs_reference(prod, ref, seed):
    kw = dict(seed=seed, rounds=3, steps=250, gpu=160, cpu=200, max_prompt=80)
    assert drv.fuzz_ops(prod, **kw) == drv.fuzz_ops(ref, **kw)


@pytest.mark.parametrize("seed", [31, 2024])
def test_fuzz_free_stacks_vs_reference(prod, ref, seed):
    """The LIFO free lists themselves (reference SlotPool::free_stack_,
    kv_manager.hpp:153-166, read from the compiled reference) after every
    op of the test_kv_manager.cpp:265-322 stream: the product's compact
    lazy stack must be the same stack, bottom to top."""
    kw = dict(seed=seed, rounds=3, steps=300, gpu=96 if seed == 2024 else 256, cpu=64 if seed == 2024 else 512,
              record_free=True)
    a, b = drv.fuzz_ops(prod, **kw), drv.fuzz_ops(ref, **kw)
    assert a == b, _first_diff(a[0], b[0])


@pytest.mark.parametrize("seed", [3, 5])
def test_fuzz_live_llama_shape(prod, ref, seed):
    """32-layer model, bigger prompts: exercises the tail-scan fetch path."""
    kw = dict(seed=seed, rounds=2, steps=150, gpu=6000, cpu=9000, model=ls.llama2_7b(), max_prompt=700,
              check_every=5)
    assert drv.fuzz_ops(prod, **kw) == drv.fuzz_ops(ref, **kw)


def test_request_views_identical(prod, ref):
    """request() (the const view engine.cpp:412 reads) entry by entry."""
    for lib_pair_seed in range(3):
        views = []
        for lib in (prod, ref):
            rnd = random.Random(lib_pair_seed)
            kv = ls.KvManager(ls.BlockPools(400, 300, 16), ls.tiny8(), lib=lib)
            ids = []
            for i in range(12):
                if kv.allocate_prefill(i, rnd.randint(1, 70), rnd.randint(0, 8)):
                    ids.append(i)
            jobs = []
            for i in ids[::2]:
                j = kv.plan_offload(i, rnd.choice([ls.HALF, ls.FULL]))
                if j and j.job_id >= 0:
                    jobs.append(j.job_id)
            for j in jobs[::2]:
                kv.complete_offload(j)
            for i in ids:
                for _ in range(rnd.randint(0, 40)):
                    if kv.needs_append(i) and not kv.append_decode_block(i):
                        break
                    kv.note_token(i)
            views.append([kv.request(i) for i in ids] + [kv.dump_table()])
        assert views[0] == views[1]


def test_release_orphans_parity(prod, ref):
    out = []
    for lib in (prod, ref):
        kv = ls.KvManager(ls.BlockPools(128, 128, 16), ls.tiny8(), lib=lib)
        kv.allocate_prefill(1, 40, 8)
        kv.allocate_prefill(2, 20, 6)
        a = kv.plan_offload(1, ls.HALF)
        b = kv.plan_offload(1, ls.FULL)
        f = kv.release(1)
        kv.check_conservation()
        kv.complete_offload(b.job_id)
        kv.allocate_prefill(3, 50, 3)
        kv.complete_offload(a.job_id)
        kv.allocate_prefill(4, 33, 5)
        out.append((f, kv.dump_table(), kv.gpu_blocks_free(), kv.cpu_blocks_free()))
    assert out[0] == out[1]
