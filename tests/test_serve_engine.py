"""Serving loop and trace / CSV formats (f4).

The product's own loop (paper_2410_00428_b200/csrc/serve_engine.cpp) with the
modelled executor must reproduce the REFERENCE engine's requests.csv byte for
byte and its summary numbers exactly, on every BASELINE.json trace
(tests/golden/engine.json, written by the compiled reference). The traces
come from the product's restated generators, so the same hashes also pin
generate_fixed / generate_sharegpt_like. Where the reference is built here,
the generators and JSONL I/O are compared with it directly."""
from __future__ import annotations

import hashlib
import json
import os

import pytest

from paper_2410_00428_b200 import layersim as ls
from paper_2410_00428_b200 import serve
from tests import _drivers as drv
from tests.golden import make_golden as mg
from tests.test_engine_dropin import FAST

SUMMARY_KEYS = ["mean_ttft", "p50_ttft", "p99_ttft", "mean_tpot", "throughput", "makespan", "d2h_jobs", "h2d_jobs",
                "d2h_bytes", "h2d_bytes", "completed", "n_rows"]


def product_trace(spec) -> serve.Trace:
    kind = spec[0]
    if kind == "single":
        return serve.Trace([0], [0.0], [spec[1]], [spec[2]])
    if kind == "fixed":
        _, n, p, o, rate, seed = spec
        return serve.generate_fixed(n, p, o, rate, seed)
    if kind == "sharegpt":
        _, n, rate, seed = spec
        return serve.generate_sharegpt_like(n, rate, seed)
    if kind == "batch":
        _, n, p, o = spec
        return serve.Trace(list(range(n)), [0.0] * n, [p] * n, [o] * n)
    rows = spec[1]
    return serve.Trace([r[0] for r in rows], [r[1] for r in rows], [r[2] for r in rows], [r[3] for r in rows])


def serve_cfg(sc, **kw) -> serve.ServeConfig:
    hw = mg.scenario_hw(sc)
    kw.setdefault("tokens_per_block", sc.get("bs", 16))
    kw.setdefault("max_batch_tokens", sc.get("max_batch_tokens", 131072))
    return serve.ServeConfig(model=getattr(ls, sc["model"])(), hw=hw, layerkv=sc["layerkv"],
                             slo_scheduler=sc.get("slo", True), gpu_blocks=sc["pools"][0], cpu_blocks=sc["pools"][1],
                             seed=sc.get("seed", 0), force_retained_layers=sc["force"],
                             invariant_checks=sc.get("invariant", False), **kw)


@pytest.fixture(scope="module")
def engine_golden():
    with open(os.path.join(os.path.dirname(__file__), "golden", "engine.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", FAST)
def test_serve_loop_matches_reference_golden(engine_golden, name):
    sc = mg.ENGINE_SCENARIOS[name]
    summary, rows, csv = serve.run(serve_cfg(sc), product_trace(sc["trace"]))
    g = engine_golden[name]
    assert csv.splitlines()[:3] == g["csv_head"]
    assert hashlib.sha256(csv.encode()).hexdigest() == g["csv_sha256"]
    assert {k: summary[k] for k in SUMMARY_KEYS} == g["summary"]


def test_trace_generators_match_reference(ref):
    for sharegpt, args in ((False, (100, 16384, 512, 1.0, 1)), (False, (7, 3, 9, 0.25, 123)),
                           (True, (150, 0, 0, 6.0, 11)), (True, (500, 0, 0, 10.0, 17))):
        want = drv.generate_trace(ref, sharegpt, *args)
        got = serve._generate(sharegpt, *args, None)
        assert (got.ids, got.arrival, got.prompt, got.output) == tuple(list(x) for x in want)


def test_jsonl_round_trip_and_errors(tmp_path):
    t = serve.generate_sharegpt_like(40, 3.0, 5)
    p = tmp_path / "t.jsonl"
    serve.save_trace(t, p)
    back, unsorted = serve.load_trace(p)
    assert not unsorted and back == t  # shortest round-trip doubles: exact
    first = p.read_text().splitlines()[0]
    rec = json.loads(first)
    assert set(rec) == {"id", "arrival_s", "prompt_tokens", "output_tokens"}

    q = tmp_path / "u.jsonl"
    q.write_text('# comment\n{"arrival_s": 2.5, "prompt_tokens": 10, "output_tokens": 3}\n\n'
                 '  {"output_tokens": 1, "prompt_tokens": 4, "arrival_s": 1}\n')
    back, unsorted = serve.load_trace(q)
    assert unsorted and back.ids == [1, 0] and back.arrival == [1.0, 2.5] and back.prompt == [4, 10]

    for body, msg in (('{"arrival_s": 1, "prompt_tokens": 2}\n', "missing field 'output_tokens'"),
                      ('{"arrival_s": 1, "prompt_tokens": 2, "output_tokens": 0}\n', "invariant violation"),
                      ('{"arrival_s": 1, "prompt_tokens": 2\n', "parse error"),
                      ('# only a comment\n', "contains no records")):
        bad = tmp_path / "bad.jsonl"
        bad.write_text(body)
        with pytest.raises(ls.LkvError, match=msg):
            serve.load_trace(bad)
    with pytest.raises(ls.LkvError, match="bad.jsonl:1"):
        bad.write_text('{"arrival_s": "x", "prompt_tokens": 2, "output_tokens": 1}\n')
        serve.load_trace(bad)


def test_reference_reads_product_jsonl(ref, tmp_path):
    """The reference's own load_trace (nlohmann json) reads what the product
    writes, and vice versa, to the same requests."""
    if not hasattr(ref.dll, "ref_load_trace"):
        pytest.skip("reference shim has no ref_load_trace")
    import ctypes as C
    t = serve.generate_sharegpt_like(25, 2.0, 9)
    p = tmp_path / "p.jsonl"
    serve.save_trace(t, p)
    n = len(t)
    ids, arr, pr, o = (C.c_int64 * n)(), (C.c_double * n)(), (C.c_int32 * n)(), (C.c_int32 * n)()
    assert ref.dll.ref_load_trace(str(p).encode(), ids, arr, pr, o, n) == n
    assert (list(ids), list(arr), list(pr), list(o)) == (t.ids, t.arrival, t.prompt, t.output)
    q = tmp_path / "r.jsonl"
    assert ref.dll.ref_save_trace(str(q).encode(), n, ids, arr, pr, o) == 0
    back, _ = serve.load_trace(q)
    assert back == t


def test_jsonl_ignores_nested_extra_fields(ref, tmp_path):
    """Extra array / object fields (metadata) are ignored, as the reference's
    nlohmann-based load_trace ignores them (workload.cpp:84-136)."""
    body = ('{"id": 3, "tags": ["a", "]}", {"x": [1, 2]}], "arrival_s": 0.5, "meta": {"k": {"z": "}"}, "n": null}, '
            '"prompt_tokens": 7, "output_tokens": 2}\n'
            '{"meta": [], "id": 4, "arrival_s": 1.25, "prompt_tokens": 9, "output_tokens": 1, "o": {}}\n')
    p = tmp_path / "nested.jsonl"
    p.write_text(body)
    back, unsorted = serve.load_trace(p)
    assert not unsorted and (back.ids, back.arrival, back.prompt, back.output) == ([3, 4], [0.5, 1.25], [7, 9], [2, 1])
    if hasattr(ref.dll, "ref_load_trace"):
        import ctypes as C
        ids, arr, pr, o = (C.c_int64 * 2)(), (C.c_double * 2)(), (C.c_int32 * 2)(), (C.c_int32 * 2)()
        assert ref.dll.ref_load_trace(str(p).encode(), ids, arr, pr, o, 2) == 2
        assert (list(ids), list(arr), list(pr), list(o)) == (back.ids, back.arrival, back.prompt, back.output)
    bad = tmp_path / "bad_nested.jsonl"
    bad.write_text('{"id": 1, "arrival_s": 0, "prompt_tokens": 2, "output_tokens": 1, "t": [1, 2\n')
    with pytest.raises(ls.LkvError, match="parse error"):
        serve.load_trace(bad)


def test_errors_are_loud():
    sc = mg.ENGINE_SCENARIOS["te_fcfs_layerkv"]
    cfg = serve_cfg(sc)
    cfg.gpu_blocks, cfg.cpu_blocks = 8, 8  # the 512-token head can never fit
    with pytest.raises(ls.SimulationError, match="can never be admitted"):
        serve.run(cfg, product_trace(sc["trace"]))
    with pytest.raises(ls.LkvError, match="arrivals not sorted"):
        serve.run(serve_cfg(sc), serve.Trace([0, 1], [1.0, 0.5], [4, 4], [2, 2]))


@pytest.fixture(scope="module")
def logs_golden():
    with open(os.path.join(os.path.dirname(__file__), "golden", "engine_logs.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", mg.TLOG_SCENARIOS)
def test_cli_logs_match_reference_golden(logs_golden, name):
    """The reference CLI's two logs (f4; SURVEY §5 tracing), byte-identical to
    the compiled reference's: transfer_log.csv (every bus transfer — submit /
    start / end, bytes, direction, all-reduce deferrals; Engine::transfer_log(),
    tools/layersim_main.cpp:96-105) and decision_log.csv (every LayerKV
    admission round that admitted or escalated — time, smallest Eq. 2 slack,
    admitted count, Half/Full plan; engine.cpp:388-390, layersim_main.cpp:107-117)."""
    sc = mg.tlog_scenario(name)
    summary, _, _, tlog, dlog = serve.run(serve_cfg(sc), product_trace(sc["trace"]), logs=True)
    for which, text in (("transfer", tlog), ("decision", dlog)):
        g = logs_golden[which][name]
        lines = text.splitlines()
        assert lines[:3] == g["head"] and len(lines) - 1 == g["rows"], which
        assert hashlib.sha256(text.encode()).hexdigest() == g["sha256"], which
    assert len(tlog.splitlines()) - 1 == summary["d2h_jobs"] + summary["h2d_jobs"]
    assert sum(1 for x in dlog.splitlines()[1:] if not x.endswith(",none")) == \
        logs_golden["decision"][name]["escalating_rows"]


@pytest.mark.parametrize("name,which", [("tlog_tp4_pcie", "transfer"), ("esc_small", "decision"),
                                        ("tlog_tp2_pcie_contended", "decision")])
def test_cli_logs_live_against_reference(ref, name, which):
    """The same files from the live reference engine, compared line by line so
    a mismatch names its row (PCIe-only TP: deferred chunks; escalations)."""
    if not hasattr(ref.dll, "ref_engine_log"):
        pytest.skip("reference shim has no ref_engine_log")
    sc = mg.tlog_scenario(name)
    want = drv.run_engine_log(ref, mg.scenario_cfg(sc), mg.make_trace(ref, sc["trace"]), which).splitlines()
    _, _, _, tlog, dlog = serve.run(serve_cfg(sc), product_trace(sc["trace"]), logs=True)
    got = (tlog if which == "transfer" else dlog).splitlines()
    assert len(got) == len(want)
    for i, (a, b) in enumerate(zip(got, want)):
        assert a == b, f"{which} row {i}: {a} != {b}"
    if which == "transfer":
        assert any(not x.endswith(",0") for x in got[1:])  # deferrals exercised
    else:
        assert any(not x.endswith(",none") for x in got[1:])  # escalations exercised


@pytest.mark.parametrize("max_time", [5.0, 20.0])
def test_wall_clock_cap_matches_reference(ref, max_time):
    """max_sim_time (engine.cpp:82-86, SURVEY §5 failure detection): a run cut
    at the cap reports completed = 0 and the same truncated requests.csv,
    summary and both CLI logs as the reference."""
    sc = dict(mg.ENGINE_SCENARIOS["te_contended"])
    trace = mg.make_trace(ref, sc["trace"])
    rcfg = mg.scenario_cfg(sc)
    rcfg.max_sim_time = max_time
    want_summary, want_csv = drv.run_engine(ref, rcfg, trace)
    want_t = drv.run_engine_log(ref, rcfg, trace, "transfer")
    want_d = drv.run_engine_log(ref, rcfg, trace, "decision")
    summary, _, csv, tlog, dlog = serve.run(serve_cfg(sc, max_time=max_time), product_trace(sc["trace"]), logs=True)
    assert want_summary["completed"] == 0 and summary["completed"] == 0
    assert {k: summary[k] for k in SUMMARY_KEYS} == want_summary
    assert csv == want_csv and tlog == want_t and dlog == want_d


def test_block_starvation_matches_reference(ref):
    """The starvation detector (engine.cpp:107-119): SURVEY §4's
    acceptance c8 run 53 — baseline policy, 16 layers, 302 GPU blocks; the
    request's 80 prompt blocks pass the never-fits check, but with its growth
    reserve (19 rows x 16 layers) it never admits, so the loop runs dry. The
    product raises the reference's exact message."""
    m = ls.ModelSpec(16, 4, 4, 32, 128, 1e8, 2)
    hw = ls.default_hardware()
    trace = ([0], [0.0], [78], [287])
    rcfg = drv.engine_cfg_struct(m, hw, layerkv=False, gpu_blocks=302, cpu_blocks=2416)
    with pytest.raises(ls.SimulationError) as want:
        drv.run_engine(ref, rcfg, trace)
    cfg = serve.ServeConfig(model=m, hw=hw, layerkv=False, gpu_blocks=302, cpu_blocks=2416)
    with pytest.raises(ls.SimulationError) as got:
        serve.run(cfg, serve.Trace(*[list(x) for x in trace]))
    assert "block starvation" in str(want.value)
    assert str(got.value) == "lkv_serve_run: " + str(want.value)  # the C ABI names its entry point


def test_serve_run_ex_sizes_and_rejects_bad_log_arguments():
    """lkv_serve_run_ex: NULL buffers size the logs (header-only logs for a
    run without transfers), a buffer without its length pointer is rejected,
    and a NULL length skips that log."""
    import ctypes as C
    from paper_2410_00428_b200 import _abi
    L = serve._lib(None)
    sc = mg.ENGINE_SCENARIOS["cfg1_x32"]  # everything retained: no transfers, one admission
    cfg, trace = serve_cfg(sc), product_trace(sc["trace"])
    n = len(trace)
    out, rows = _abi.ServeSummaryC(), (_abi.ServeRowC * n)()
    tl, dl = C.c_size_t(), C.c_size_t()
    L.call("lkv_serve_run_ex", C.byref(cfg.c()), n, *trace.arrays(), C.byref(out), rows, n, None, 0, C.byref(tl),
           None, 0, C.byref(dl))
    assert tl.value == len("submit_s,start_s,end_s,bytes,direction,deferrals\n")
    assert dl.value == len("time_s,min_budget_s,admitted,offload_plan\n") + len("0,inf,1,none\n")
    buf = C.create_string_buffer(64)
    with pytest.raises(ls.LkvError, match="invalid argument"):
        L.call("lkv_serve_run_ex", C.byref(cfg.c()), n, *trace.arrays(), C.byref(out), rows, n, buf, 64, None,
               None, 0, None)
    L.call("lkv_serve_run_ex", C.byref(cfg.c()), n, *trace.arrays(), C.byref(out), rows, n, None, 0, None, None, 0,
           None)
    assert out.completed == 1
