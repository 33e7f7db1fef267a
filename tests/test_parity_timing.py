"""Cost model, PcieBus and schedule_prefill_span: bit-exact (==, not approx)
with the reference, plus the reference's own unit assertions
(proj/tests/test_cost_model.cpp, test_interconnect.cpp, test_engine.cpp:175-223)."""
import math
import random

import pytest

from paper_2410_00428_b200 import layersim as ls
from tests._drivers import Rng


def pcie2():
    return ls.HardwareSpec(1e14, 8.64e11, 3.2e10, False, 2, 48e9, 0.9)


def single():
    return ls.HardwareSpec(1e14, 8.64e11, 3.2e10, False, 1, 48e9, 0.9)


def rand_model(r):
    L = r.randint(1, 127)
    kvh = r.choice([1, 2, 4, 8, 16, 32])
    g = r.choice([1, 2, 4, 8])
    d = r.choice([64, 128])
    return ls.ModelSpec(L, kvh * g, kvh, d, kvh * g * d, r.uniform(1e8, 1e11), r.choice([1, 2, 4]))


def rand_hw(r):
    return ls.HardwareSpec(r.uniform(1e13, 3e15), r.uniform(5e11, 8e12), r.uniform(1e9, 1e11), r.random() < 0.5,
                           r.randint(1, 8), r.uniform(16e9, 200e9), r.uniform(0.5, 1.0))


def test_cost_functions_bit_exact(prod, ref):
    r = random.Random(5)
    for _ in range(300):
        m, hw = rand_model(r), rand_hw(r)
        p = ls.CostParams(r.uniform(0.5, 2), r.uniform(0.5, 2), r.uniform(0.5, 2), r.uniform(0.1, 0.9))
        s = r.randint(1, 200000)
        for fn, args in ((ls.prefill_time, (m, hw, p, s)), (ls.decode_step_time, (m, hw, p, s)),
                         (ls.allreduce_time, (m, hw, s)), (ls.min_retained_layers, (m, hw, p, s)),
                         (ls.offload_time, (m, hw, p, s, r.randint(0, m.n_layers))),
                         (ls.kv_bytes_per_token_layer, (m,))):
            assert fn(*args, lib=prod) == fn(*args, lib=ref)


def test_cost_model_worked_values(prod):  # test_cost_model.cpp:79-86 and :45-66
    assert ls.kv_bytes_per_token_layer(ls.llama2_7b(), lib=prod) == 16384
    assert ls.kv_bytes_per_token_layer(ls.llama3_8b_gqa(), lib=prod) == 4096
    t = ls.prefill_time(ls.llama2_7b(), ls.default_hardware(), ls.CostParams(), 1024, lib=prod)
    assert f"{t:.9g}" == "0.143445899"  # BASELINE.md config 1 TTFT
    with pytest.raises(ls.DomainError):
        ls.offload_time(ls.llama2_7b(), ls.default_hardware(), ls.CostParams(), 10, 33, lib=prod)


def test_min_retained_layers_minimal_and_monotone(prod):  # test_cost_model.cpp:131-167
    m, hw, p = ls.llama2_7b(), ls.default_hardware(), ls.CostParams()
    prev = m.n_layers
    for s in (64, 128, 256, 512, 1024, 2048, 4096, 16384):
        x = ls.min_retained_layers(m, hw, p, s, lib=prod)
        assert ls.offload_time(m, hw, p, s, m.n_layers - x, lib=prod) <= ls.prefill_time(m, hw, p, s, lib=prod)
        if x > 0:
            assert ls.offload_time(m, hw, p, s, m.n_layers - x + 1, lib=prod) > ls.prefill_time(m, hw, p, s, lib=prod)
        assert x <= prev
        prev = x


# ---------------------------------------------------------------- PcieBus
def test_bus_unit_cases(prod):  # test_interconnect.cpp:29-93
    bus = ls.PcieBus(lib=prod)
    s = bus.submit_transfer(0.0, ls.D2H, 5.0, 1 << 20, single())
    assert s.completion == 5.0 and s.chunks == 0 and bus.busy_until() == 0.0
    bus = ls.PcieBus(lib=prod)
    s = bus.submit_transfer(1024.0 ** 3, ls.D2H, 1.0, 16 * 1024 * 1024, single())
    assert s.start == 1.0 and math.isclose(s.completion, 1.033554432, rel_tol=1e-12)
    assert s.chunks == 64 and s.deferrals == 0
    bus = ls.PcieBus(lib=prod)
    a = bus.submit_transfer(3.2e8, ls.D2H, 0.0, 1 << 24, single())
    b = bus.submit_transfer(3.2e8, ls.H2D, 0.001, 1 << 24, single())
    assert math.isclose(a.completion, 0.01, rel_tol=1e-12) and math.isclose(b.start, 0.01, rel_tol=1e-12)
    bus = ls.PcieBus(0.5, lib=prod)
    bus.register_allreduce(0.0, 0.010, pcie2())
    assert bus.allreduce_active(0.005)
    s = bus.submit_transfer(3.2e8, ls.D2H, 0.0, 1 << 24, pcie2())
    assert math.isclose(s.start, 0.010, rel_tol=1e-9) and s.deferrals > 1
    assert math.isclose(s.completion, 0.020, rel_tol=1e-9)
    nv = pcie2()
    nv.nvlink = True
    bus = ls.PcieBus(lib=prod)
    bus.register_allreduce(0.0, 1.0, nv)
    bus.register_allreduce(0.0, 1.0, single())
    assert bus.allreduce_busy_until() == 0.0


def test_bus_window_union_and_midchunk(prod):  # test_interconnect.cpp:95-122
    bus = ls.PcieBus(lib=prod)
    bus.register_allreduce(0.0, 0.005, pcie2())
    bus.register_allreduce(0.003, 0.005, pcie2())
    assert math.isclose(bus.allreduce_busy_until(), 0.008, rel_tol=1e-12)
    s = bus.submit_transfer(3.2e7, ls.D2H, 0.001, 1 << 25, pcie2())
    assert math.isclose(s.start, 0.008, rel_tol=1e-9)
    bus = ls.PcieBus(lib=prod)
    bus.enable_history(True)
    bus.submit_transfer(16.0 * 1024 * 1024, ls.D2H, 0.0, 1 << 24, pcie2())
    end = bus.busy_until()
    bus.register_allreduce(end / 2.0, 0.001, pcie2())
    assert math.isclose(bus.allreduce_busy_until(), end + 0.001, rel_tol=1e-12)


@pytest.mark.parametrize("seed", [2024, 7, 11])
def test_bus_disjointness_property_bit_exact(prod, ref, seed):
    """test_interconnect.cpp:136-164 generator; product == reference for every
    schedule, chunk and window, and chunks never overlap windows."""
    outs = []
    for lib in (prod, ref):
        rng = Rng(seed)
        hw = pcie2()
        rounds = []
        for _ in range(20):
            bus = ls.PcieBus(0.25 + 0.5 * rng.uniform01(), lib=lib)
            bus.enable_history(True)
            t, scheds = 0.0, []
            for _span in range(15):
                dur = 0.002 + 0.004 * rng.uniform01()
                for _w in range(rng.uniform_below(3)):
                    bus.register_allreduce(t + dur * rng.uniform01(), 0.002 * rng.uniform01(), hw)
                submit = t
                for _j in range(rng.uniform_below(3)):
                    submit += dur * rng.uniform01() / 2.0
                    scheds.append(bus.submit_transfer(1e5 + rng.uniform01() * 5e7, ls.D2H, submit, 1 << 22, hw))
                t += dur
            chunks, wins = bus.chunk_history(), bus.allreduce_windows()
            for c0, c1, _ in chunks:
                for w0, w1, _ in wins:
                    assert c1 <= w0 + 1e-12 or w1 <= c0 + 1e-12
            rounds.append((scheds, chunks, wins))
        outs.append(rounds)
    assert outs[0] == outs[1]


def test_bus_random_ops_bit_exact(prod, ref):
    r = random.Random(77)
    ops = []
    t = 0.0
    for _ in range(400):
        t += r.random() * 0.003
        if r.random() < 0.4:
            ops.append(("ar", t, r.random() * 0.004))
        else:
            ops.append(("tx", r.random() * 8e7, r.randint(0, 1), t, r.choice([1 << 20, 1 << 24])))
    res = []
    for lib in (prod, ref):
        bus = ls.PcieBus(0.37, lib=lib)
        out = []
        for op in ops:
            if op[0] == "ar":
                bus.register_allreduce(op[1], op[2], pcie2())
            else:
                out.append(bus.submit_transfer(op[1], op[2], op[3], op[4], pcie2()))
            out.append((bus.busy_until(), bus.allreduce_busy_until()))
        res.append(out)
    assert res[0] == res[1]


# ---------------------------------------------------------------- prefill span
def test_prefill_span_bit_exact_and_overlap_invariant(prod, ref):
    """test_engine.cpp:175-203: completion never delayed by the transfers;
    one job per offloaded layer; every time == reference."""
    cost = ls.CostParams()
    for seed in range(30):
        rng = Rng(seed)
        L = 8 + rng.uniform_below(72)
        H = 8 + rng.uniform_below(56)
        m = ls.ModelSpec(L, H, H, 128, H * 128, 7.0e9, 2)
        hw = ls.default_hardware()
        hw.pcie_bandwidth = 1e9 + rng.uniform01() * 6e10
        hw.n_gpus = 1 + rng.uniform_below(4)
        hw.nvlink = rng.uniform_below(2) == 0
        prompt = 64 + rng.uniform_below(8192)
        x = ls.min_retained_layers(m, hw, cost, prompt, lib=prod)
        plan = ls.layer_placement(L, x, lib=prod)
        got = []
        for lib in (prod, ref):
            on = ls.schedule_prefill_span(m, hw, cost, ls.PcieBus(cost.delta, lib=lib), plan.offloaded, prompt,
                                          1.0, 1 << 24, True, lib=lib)
            off = ls.schedule_prefill_span(m, hw, cost, ls.PcieBus(cost.delta, lib=lib), plan.offloaded, prompt,
                                           1.0, 1 << 24, False, lib=lib)
            assert on[0] == off[0] and len(on[1]) == len(plan.offloaded) and off[1] == []
            got.append(on)
        assert got[0] == got[1]


def test_prefill_span_full_offload_times(prod):  # test_engine.cpp:205-223
    m, hw, p = ls.llama2_7b(), ls.default_hardware(), ls.CostParams()
    T = ls.prefill_time(m, hw, p, 2048, lib=prod)
    bus = ls.PcieBus(lib=prod)
    comp, jobs = ls.schedule_prefill_span(m, hw, p, bus, list(range(32)), 2048, 0.0, 1 << 24, True, lib=prod)
    assert len(jobs) == 32 and comp == T
    # jobs are submitted at (i+1) T / 32 and serialise on the bus
    assert math.isclose(jobs[0].start, T / 32, rel_tol=1e-9)
