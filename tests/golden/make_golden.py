"""Generate the committed golden fixtures from the COMPILED REFERENCE.

Run here (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
The fixtures let the GPU box, where the reference sources do not exist, check
the product against reference outputs. Every value below is produced by the
reference's own C++ (oracle/_ref/libref_layersim.so), never by the product.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from paper_2410_00428_b200 import layersim as ls  # noqa: E402
from tests import _drivers as drv  # noqa: E402

ENGINE_SCENARIOS = {
    # one request {0, 1024, 65}, pools {200000, 800000}
    **{f"cfg1_x{x}": dict(model="llama2_7b", pools=(200000, 800000), layerkv=True, force=x,
                          trace=("single", 1024, 65)) for x in (32, 16, 0)},
    # 48 GB budget (113043 blocks), fixed(100, ctx, 512, 1 req/s, seed 1)
    **{f"cfg2_{pol}_{ctx}": dict(model="llama2_7b", pools=(113043, 904344), layerkv=(pol == "layerkv"),
                                 force=-1, seed=1, trace=("fixed", 100, ctx, 512, 1.0, 1))
       for ctx in (128, 1024, 2048, 4096, 16384) for pol in ("baseline", "layerkv")},
    # proj/tests/test_engine.cpp scenarios
    "te_determinism_layerkv": dict(model="llama2_7b", pools=(6000, 48000), layerkv=True, force=-1, seed=7,
                                   trace=("sharegpt", 150, 6.0, 11)),
    "te_determinism_baseline": dict(model="llama2_7b", pools=(6000, 48000), layerkv=False, force=-1, seed=7,
                                    trace=("sharegpt", 150, 6.0, 11)),
    "te_contended": dict(model="llama2_7b", pools=(3000, 24000), layerkv=True, force=-1, seed=7, invariant=True,
                         trace=("sharegpt", 120, 10.0, 17)),
    "te_fcfs_layerkv": dict(model="llama2_7b", pools=(1800, 7200), layerkv=True, force=-1, seed=7, invariant=True,
                            trace=("list", [(0, 0.0, 512, 64), (1, 0.1, 768, 8), (2, 0.2, 16, 8)])),
    "te_slo_ablation": dict(model="llama2_7b", pools=(200000, 800000), layerkv=True, slo=False, force=-1, seed=7,
                            trace=("fixed", 60, 4096, 64, 2.0, 29)),
    # small escalation case for the device-executed serving loop (3 Half/Full escalations)
    "esc_small": dict(model="llama2_7b", pools=(600, 20000), layerkv=True, force=-1, seed=3, invariant=True,
                      trace=("sharegpt", 12, 20.0, 17)),
    # 70B GQA, TP8 over NVLink, half retained (config 4 shape, 4k + 64)
    "cfg4_tp8": dict(model="llama31_70b_gqa", tp=8, nvlink=True, pools=(2000000, 16000000), layerkv=True, force=40,
                     trace=("single", 4096, 65)),
}


def make_trace(lib, spec):
    kind = spec[0]
    if kind == "single":
        return [0], [0.0], [spec[1]], [spec[2]]
    if kind == "fixed":
        _, n, p, o, rate, seed = spec
        return drv.generate_trace(lib, False, n, p, o, rate, seed)
    if kind == "sharegpt":
        _, n, rate, seed = spec
        return drv.generate_trace(lib, True, n, 0, 0, rate, seed)
    rows = spec[1]
    return [r[0] for r in rows], [r[1] for r in rows], [r[2] for r in rows], [r[3] for r in rows]


def scenario_cfg(sc):
    model = getattr(ls, sc["model"])()
    hw = ls.default_hardware()
    hw.n_gpus = sc.get("tp", 1)
    hw.nvlink = sc.get("nvlink", False)
    return drv.engine_cfg_struct(model, hw, layerkv=sc["layerkv"], slo=sc.get("slo", True),
                                 gpu_blocks=sc["pools"][0], cpu_blocks=sc["pools"][1], seed=sc.get("seed", 0),
                                 force_retained=sc["force"], invariant_checks=sc.get("invariant", False))


def engine_goldens(lib):
    out = {}
    for name, sc in ENGINE_SCENARIOS.items():
        trace = make_trace(lib, sc["trace"])
        summary, csv = drv.run_engine(lib, scenario_cfg(sc), trace)
        out[name] = {"summary": summary, "csv_sha256": hashlib.sha256(csv.encode()).hexdigest(),
                     "csv_head": csv.splitlines()[:3]}
        print(name, summary["p50_ttft"], summary["p99_ttft"], summary["mean_tpot"], flush=True)
    return out


def kv_goldens(lib):
    m = ls.llama2_7b()
    res = {}
    for x in (0, 16, 32):
        kv = ls.KvManager(ls.BlockPools(200000, 800000, 16), m, lib=lib)
        kv.allocate_prefill(0, 1024, x)
        h1 = format(kv.dump_hash(), "016x")
        for _ in range(64):
            if kv.needs_append(0):
                kv.append_decode_block(0)
            kv.note_token(0)
        res[f"cfg1_x{x}"] = {"after_prefill": h1, "after_64": format(kv.dump_hash(), "016x"),
                             "gpu_free": kv.gpu_blocks_free(), "cpu_free": kv.cpu_blocks_free(),
                             "fetch": [(j.layer, j.bytes) for j in kv.plan_decode_fetch(0)]}
    fuzz = drv.fuzz_ops(lib)  # Rng(31), 10 x 300: test_kv_manager.cpp:265-322
    res["fuzz_rng31"] = {"digest": drv.trace_digest(fuzz), "round0": fuzz[0]}
    fuzz2 = drv.fuzz_ops(lib, seed=2024, rounds=6, steps=400, gpu=96, cpu=64, max_prompt=48)
    res["fuzz_tight_2024"] = {"digest": drv.trace_digest(fuzz2), "round0": fuzz2[0]}
    return res


def main():
    oracle.build()
    lib = oracle.ref_lib()
    kv = kv_goldens(lib)
    with open(os.path.join(HERE, "kv_manager.json"), "w") as f:
        json.dump(kv, f)
    eng = engine_goldens(lib)
    with open(os.path.join(HERE, "engine.json"), "w") as f:
        json.dump(eng, f, indent=1)


if __name__ == "__main__":
    main()
