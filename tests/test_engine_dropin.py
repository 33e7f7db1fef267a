"""Drop-in proof: the reference event loop (proj/src/engine.cpp, unmodified,
compiled against the product headers and linked with the product KvManager,
PcieBus and cost model — oracle/_ref/libhybrid_layersim.so) produces
byte-identical requests.csv and identical TTFT p50/p99, TPOT and transfer
totals to the pure reference, on the BASELINE.json configs' traces."""
import hashlib

import pytest

from tests import _drivers as drv
from tests.golden import make_golden as mg

FAST = ["cfg1_x32", "cfg1_x16", "cfg1_x0", "cfg2_baseline_128", "cfg2_layerkv_128", "cfg2_baseline_1024",
        "cfg2_layerkv_1024", "cfg2_baseline_2048", "cfg2_layerkv_2048", "te_determinism_layerkv",
        "te_determinism_baseline", "te_contended", "te_fcfs_layerkv", "cfg4_tp8", "cfg2_baseline_4096",
        "cfg2_layerkv_4096", "te_slo_ablation", "cfg2_baseline_16384", "cfg2_layerkv_16384", "esc_small",
        # round 2: config 2 at 512 / 8192, config 3 (8B GQA, B200 spec) at batch 64 / 24 / 4, config 4 at
        # TP 1/2/4/8 on the B200 spec, config 5's block sizes 16/32/64
        "cfg2_baseline_512", "cfg2_layerkv_512", "cfg2_baseline_8192", "cfg2_layerkv_8192", "cfg3_b64", "cfg3_b24",
        "cfg3_b4", *[f"cfg4_b200_tp{tp}" for tp in (1, 2, 4, 8)],
        *[f"cfg5_7b_4k_k{k}_bs{bs}" for k in (1, 16, 32) for bs in (16, 32, 64)],
        *[f"cfg5_70b_128k_tp8_bs{bs}" for bs in (16, 32, 64)]]


def _run(lib, name):
    sc = mg.ENGINE_SCENARIOS[name]
    trace = mg.make_trace(lib, sc["trace"])
    return drv.run_engine(lib, mg.scenario_cfg(sc), trace)


@pytest.mark.parametrize("name", FAST)
def test_hybrid_engine_matches_reference_golden(hybrid, golden, name):
    summary, csv = _run(hybrid, name)
    g = golden["engine"][name]
    assert hashlib.sha256(csv.encode()).hexdigest() == g["csv_sha256"]
    assert summary == g["summary"]


def test_golden_pins_baseline_md(golden):
    """The engine goldens reproduce the numbers printed in BASELINE.md §2."""
    e = golden["engine"]
    for x, tpot in ((32, "0.0168441967"), (16, "0.0173846127"), (0, "0.0178293504")):
        s = e[f"cfg1_x{x}"]["summary"]
        assert f"{s['p50_ttft']:.9g}" == "0.143445899" and f"{s['mean_tpot']:.9g}" == tpot
    assert e["cfg1_x0"]["summary"]["d2h_jobs"] == 32 and e["cfg1_x0"]["summary"]["d2h_bytes"] == 536870912
    assert e["cfg1_x0"]["summary"]["h2d_jobs"] == 2048 and e["cfg1_x0"]["summary"]["h2d_bytes"] == 35416702976
    assert e["cfg1_x16"]["summary"]["h2d_bytes"] == 17708351488
    s = e["cfg2_layerkv_16384"]["summary"]
    assert f"{s['p50_ttft']:.4g}" == "3827" and round(s["p99_ttft"], -1) == 11150
    s = e["cfg2_baseline_2048"]["summary"]
    assert f"{s['p50_ttft']:.3g}" == "10" and f"{s['p99_ttft']:.4g}" == "34.76"
    s = e["cfg2_layerkv_8192"]["summary"]
    assert f"{s['p50_ttft']:.4g}" == "111.5" and f"{s['p99_ttft']:.4g}" == "3736" and f"{s['mean_tpot']:.4g}" == "3.991"
    assert round(s["d2h_bytes"] / 1e9) == 406 and round(s["h2d_bytes"] / 1e12, 1) == 213.8


def test_golden_pins_survey_app_b_configs_3_to_5(golden):
    """SURVEY App. B (the compiled reference on the B200-like spec): config 3's TTFT / TPOT / job
    counts, config 4's TTFT at TP 1/2/4/8 with TP-independent bytes, and config 5's job bytes
    independent of the block size."""
    e = golden["engine"]
    s = e["cfg3_b64"]["summary"]
    assert f"{s['p50_ttft']:.4g}" == "12.39" and f"{s['p99_ttft']:.4g}" == "24.79"
    assert f"{s['mean_tpot']:.4g}" == "5.195"
    assert (s["d2h_jobs"], s["h2d_jobs"]) == (2017, 131072)
    assert round(s["d2h_bytes"] / 1e9, 1) == 274.9 and round(s["h2d_bytes"] / 1e12, 1) == 17.6
    # every request of the reduced batches is fully offloaded too (4 GiB of KV each)
    for n in (4, 24):
        assert e[f"cfg3_b{n}"]["summary"]["d2h_bytes"] == n * 32 * 32768 * 4096
    ttft = [e[f"cfg4_b200_tp{tp}"]["summary"]["p50_ttft"] for tp in (1, 2, 4, 8)]
    assert [f"{t:.4g}" for t in ttft] == ["0.4189", "0.2094", "0.1047", "0.05236"]
    byts = {(e[f"cfg4_b200_tp{tp}"]["summary"]["d2h_bytes"], e[f"cfg4_b200_tp{tp}"]["summary"]["h2d_bytes"])
            for tp in (1, 2, 4, 8)}
    assert byts == {(671088640.0, 43279974400.0)}
    keys = ("d2h_jobs", "h2d_jobs", "d2h_bytes", "h2d_bytes", "p50_ttft", "mean_tpot")
    for stem in [f"cfg5_7b_4k_k{k}" for k in (1, 16, 32)] + ["cfg5_70b_128k_tp8"]:
        got = {tuple(e[f"{stem}_bs{bs}"]["summary"][k] for k in keys) for bs in (16, 32, 64)}
        assert len(got) == 1, (stem, got)
    s = e["cfg5_70b_128k_tp8_bs16"]["summary"]
    assert round(s["d2h_bytes"] / 1e9, 2) == 42.95 and round(s["h2d_bytes"] / 1e9, 1) == 343.6
