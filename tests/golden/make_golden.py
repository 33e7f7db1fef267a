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

B200_HW = dict(flops=1.3814e15, hbm_bandwidth=6.5367e12, pcie_bandwidth=5.5e10, nvlink=True, n_gpus=1,
               gpu_mem=180e9, kv_reserve_fraction=0.9)  # SURVEY App. B's B200-like spec for configs 3-5


def _pools(model, bs, hw=None, n_gpus=1):
    """reference pool_size_from_hardware (kv_manager.cpp:10-32) at block size `bs`, restated in
    Python so the scenario table is importable without a library (fixed numbers, pinned by
    tests/test_kv_manager.py against both libraries)."""
    import math
    m = getattr(ls, model)()
    h = dict(B200_HW if hw == "b200" else dict(gpu_mem=48e9, kv_reserve_fraction=0.9))
    weight = m.n_param * m.f_precision
    act = 2.0 * 16384 * m.hidden * m.f_precision * 4.0
    kvb = (h["gpu_mem"] * n_gpus - weight - act) * h["kv_reserve_fraction"]
    g = int(math.floor(kvb / (bs * 2 * m.n_kv_heads * m.d_head * m.f_precision)))
    return g, int(math.floor(g * 8.0))


CFG5_POOLS_7B = {bs: _pools("llama2_7b", bs) for bs in (16, 32, 64)}
CFG5_POOLS_70B = {bs: _pools("llama31_70b_gqa", bs, "b200", 8) for bs in (16, 32, 64)}

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
    # the same on the B200-like spec at TP 1/2/4/8: the cost model's prefill/decode times scale with TP
    # (cost_model.cpp:39-44, 73-79; TTFT 0.4189/0.2094/0.1047/0.05236 s), the job bytes do not
    **{f"cfg4_b200_tp{tp}": dict(model="llama31_70b_gqa", hw="b200", tp=tp, nvlink=True, pools=(2000000, 16000000),
                                 layerkv=True, force=40, trace=("single", 4096, 65)) for tp in (1, 2, 4, 8)},
    # config 2 at the two remaining BASELINE.md contexts
    **{f"cfg2_{pol}_{ctx}": dict(model="llama2_7b", pools=(113043, 904344), layerkv=(pol == "layerkv"),
                                 force=-1, seed=1, trace=("fixed", 100, ctx, 512, 1.0, 1))
       for ctx in (512, 8192) for pol in ("baseline", "layerkv")},
    # config 3: Llama-3-8B GQA (no preset: override), B200-like HardwareSpec, pools from
    # pool_size_from_hardware(180 GB, max_input_tokens 32768); 64 x {0.0, 32768, 65}; max_batch_tokens
    # admits the whole batch (p50/p99 TTFT 12.39/24.79 s, 2017 D2H / 131072 H2D jobs)
    "cfg3_b64": dict(model="llama3_8b_gqa", hw="b200", pools=(2221882, 17775056), layerkv=True, force=-1,
                     max_batch_tokens=64 * (32768 + 65), trace=("batch", 64, 32768, 65)),
    # the same at the batches device runs use (host RAM holds 24 x 4.3 GB CPU-resident), with the GPU pool
    # scaled by batch/64 so the memory pressure, and hence every request's full offload, is the same
    **{f"cfg3_b{n}": dict(model="llama3_8b_gqa", hw="b200", pools=(2221882 * n // 64, 2221882 * n // 64 * 8),
                          layerkv=True, force=-1, max_batch_tokens=n * (32768 + o), trace=("batch", n, 32768, o))
       for n, o in ((4, 9), (24, 3))},
    # config 5: block sizes 16/32/64 on the same memory (pools from pool_size_from_hardware at each bs);
    # the reference's job bytes are token-exact and must not depend on bs (kv_manager.cpp:255-257, 297-299)
    **{f"cfg5_7b_4k_k{k}_bs{bs}": dict(model="llama2_7b", pools=CFG5_POOLS_7B[bs], bs=bs, layerkv=True,
                                       force=32 - k, trace=("single", 4096, 65))
       for k in (1, 16, 32) for bs in (16, 32, 64)},
    **{f"cfg5_70b_128k_tp8_bs{bs}": dict(model="llama31_70b_gqa", hw="b200", tp=8, nvlink=True,
                                         pools=CFG5_POOLS_70B[bs], bs=bs, layerkv=True, force=0,
                                         max_batch_tokens=131072 + 9, trace=("single", 131072, 9))
       for bs in (16, 32, 64)},
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
    if kind == "batch":  # n requests arriving together at t = 0
        _, n, p, o = spec
        return list(range(n)), [0.0] * n, [p] * n, [o] * n
    rows = spec[1]
    return [r[0] for r in rows], [r[1] for r in rows], [r[2] for r in rows], [r[3] for r in rows]


def scenario_hw(sc) -> ls.HardwareSpec:
    hw = ls.HardwareSpec(**B200_HW) if sc.get("hw") == "b200" else ls.default_hardware()
    hw.n_gpus = sc.get("tp", 1)
    hw.nvlink = sc.get("nvlink", hw.nvlink)
    return hw


def scenario_cfg(sc):
    model = getattr(ls, sc["model"])()
    return drv.engine_cfg_struct(model, scenario_hw(sc), layerkv=sc["layerkv"], slo=sc.get("slo", True),
                                 gpu_blocks=sc["pools"][0], cpu_blocks=sc["pools"][1], seed=sc.get("seed", 0),
                                 force_retained=sc["force"], invariant_checks=sc.get("invariant", False),
                                 tpb=sc.get("bs", 16), max_batch_tokens=sc.get("max_batch_tokens", 131072))


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


# transfer_log.csv / decision_log.csv goldens (f4, SURVEY §5 tracing): scenarios of ENGINE_SCENARIOS, plus PCIe-only
# tensor parallelism (nvlink off), where all-reduce windows defer chunks and
# the deferrals column is non-zero (interconnect.cpp check-and-delay).
TLOG_SCENARIOS = ["cfg1_x32", "cfg1_x0", "cfg2_layerkv_1024", "cfg2_baseline_1024", "te_contended", "esc_small",
                  "cfg4_b200_tp4", "cfg5_7b_4k_k16_bs32", "tlog_tp4_pcie", "tlog_tp2_pcie_contended"]
TLOG_EXTRA = {
    "tlog_tp4_pcie": {"model": "llama31_70b_gqa", "tp": 4, "nvlink": False, "pools": (2000000, 16000000),
                      "layerkv": True, "force": 40, "trace": ("fixed", 6, 2048, 17, 4.0, 5)},
    "tlog_tp2_pcie_contended": {"model": "llama2_7b", "tp": 2, "nvlink": False, "pools": (3000, 24000),
                                "layerkv": True, "force": -1, "seed": 7, "trace": ("sharegpt", 40, 10.0, 17)},
}


def tlog_scenario(name):
    return TLOG_EXTRA[name] if name in TLOG_EXTRA else ENGINE_SCENARIOS[name]


def tlog_goldens(lib):
    out = {"transfer": {}, "decision": {}}
    for name in TLOG_SCENARIOS:
        sc = tlog_scenario(name)
        for which in ("transfer", "decision"):
            csv = drv.run_engine_log(lib, scenario_cfg(sc), make_trace(lib, sc["trace"]), which)
            lines = csv.splitlines()
            g = {"sha256": hashlib.sha256(csv.encode()).hexdigest(), "rows": len(lines) - 1, "head": lines[:3]}
            if which == "transfer":
                g["deferred_rows"] = sum(1 for x in lines[1:] if not x.endswith(",0"))
            else:
                g["escalating_rows"] = sum(1 for x in lines[1:] if not x.endswith(",none"))
            out[which][name] = g
        print(name, out["transfer"][name]["rows"], out["decision"][name]["rows"], flush=True)
    return out


def main():
    import sys
    if sys.argv[1:] == ["logs"]:
        oracle.build()
        with open(os.path.join(HERE, "engine_logs.json"), "w") as f:
            json.dump(tlog_goldens(oracle.ref_lib()), f, indent=1)
        return
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
