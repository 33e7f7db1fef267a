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
        "cfg2_layerkv_4096", "te_slo_ablation", "cfg2_baseline_16384", "cfg2_layerkv_16384", "esc_small"]


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
