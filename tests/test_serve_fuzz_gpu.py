"""Serving loop on the GPU against the live compiled reference (SURVEY §8f
f1 x f3): random ShareGPT-like traces under small pools (so the SLO
scheduler escalates and most layers are offloaded), executed by the device
(every prefill, escalation and decode iteration moves real bytes; with and
without the tiered host memory), must give the reference Engine::run's
requests.csv byte for byte and bit-exact KV for every request.

Needs a GPU and oracle/_ref (built in the container, shipped with the repo
to the GPU box); skips otherwise."""
from __future__ import annotations

import pytest

from paper_2410_00428_b200 import layersim as ls
from paper_2410_00428_b200 import serve
from tests import _drivers as drv

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,gpu_blocks,pinned", [(101, 500, 0), (102, 700, 2500), (103, 400, 0), (104, 900, 4000),
                                                     (105, 600, 3000)])
def test_device_virtual_random_traces_match_live_reference(ref, seed, gpu_blocks, pinned):
    model = ls.llama2_7b()
    hw = ls.default_hardware()
    cpu_blocks = 20000
    ids, arr, p, o = drv.generate_trace(ref, True, 10, 0, 0, 20.0, seed)
    want_summary, want_csv = drv.run_engine(
        ref, drv.engine_cfg_struct(model, hw, gpu_blocks=gpu_blocks, cpu_blocks=cpu_blocks, seed=seed,
                                   invariant_checks=True), (ids, arr, p, o))
    cfg = serve.ServeConfig(model=model, hw=hw, gpu_blocks=gpu_blocks, cpu_blocks=cpu_blocks, seed=seed,
                            invariant_checks=True, executor="device-virtual", dense_gemms=False,
                            prefill_attention=False, verify_kv=True, pinned_frames=pinned)
    summary, rows, csv = serve.run(cfg, serve.Trace(ids, arr, p, o))
    assert csv == want_csv
    assert summary["completed"] == want_summary["completed"]
    assert summary["requests_verified"] == len(ids)
    assert summary["kv_words_mismatched"] == 0
