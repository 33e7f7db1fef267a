"""Serving-loop soak on the GPU against the live compiled reference
(development aid; the pytest version is tests/test_serve_fuzz_gpu.py):
N random ShareGPT-like traces, pools and tier sizes drawn per seed,
device-virtual execution vs the reference Engine::run: requests.csv, the
CLI's transfer_log.csv / decision_log.csv, and every request's KV bytes.

  python scripts/serve_soak.py [--n 24] [--seed0 1000]

One JSON line per trace; exit status 1 on any mismatch."""
import argparse
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2410_00428_b200 import layersim as ls  # noqa: E402
from paper_2410_00428_b200 import serve  # noqa: E402
from tests import _drivers as drv  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=24)
    p.add_argument("--seed0", type=int, default=1000)
    p.add_argument("--models", action="store_true", help="draw 7B / 8B GQA / 70B TP8 shards and block sizes 16-64")
    a = p.parse_args()
    ref = oracle.ref_lib()
    bad = 0
    for k in range(a.n):
        seed = a.seed0 + k
        rng = random.Random(seed)
        n_req = rng.choice([6, 10, 16])
        rate = rng.choice([5.0, 20.0, 50.0])
        gpu_blocks = rng.choice([300, 500, 800, 1500])
        cpu_blocks = 20000
        pinned = rng.choice([0, 0, 2000, 4000])
        layerkv = rng.random() < 0.85
        kind = rng.choice(["7b", "7b", "8b_gqa", "70b_tp8"]) if a.models else "7b"
        bs = rng.choice([16, 16, 32, 64]) if a.models else 16
        hw = ls.default_hardware()
        tp_rank = 0
        if kind == "7b":
            model = ls.llama2_7b()
        elif kind == "8b_gqa":
            model = ls.llama3_8b_gqa()
        else:  # 70B GQA sharded by KV head over 8 GPUs: this GPU runs one shard
            model = ls.llama31_70b_gqa()
            hw = ls.HardwareSpec(hw.flops, hw.hbm_bandwidth, hw.pcie_bandwidth, True, 8, hw.gpu_mem,
                                 hw.kv_reserve_fraction)
            tp_rank = rng.randrange(8)
        ids, arr, pr, out = drv.generate_trace(ref, True, n_req, 0, 0, rate, seed)
        t0 = time.perf_counter()
        try:
            rcfg = drv.engine_cfg_struct(model, hw, layerkv=layerkv, gpu_blocks=gpu_blocks, cpu_blocks=cpu_blocks,
                                         seed=seed, tpb=bs, invariant_checks=True)
            ws, wcsv = drv.run_engine(ref, rcfg, (ids, arr, pr, out))
            wt = drv.run_engine_log(ref, rcfg, (ids, arr, pr, out), "transfer")
            wd = drv.run_engine_log(ref, rcfg, (ids, arr, pr, out), "decision")
        except ls.SimulationError as e:  # the reference itself rejects the case: skip it
            print(json.dumps({"seed": seed, "skipped": str(e)}), flush=True)
            continue
        cfg = serve.ServeConfig(model=model, hw=hw, layerkv=layerkv, gpu_blocks=gpu_blocks, cpu_blocks=cpu_blocks,
                                seed=seed, invariant_checks=True, executor="device-virtual", dense_gemms=False,
                                prefill_attention=False, verify_kv=True, pinned_frames=pinned,
                                tokens_per_block=bs, tp_rank=tp_rank)
        s, rows, csv, tlog, dlog = serve.run(cfg, serve.Trace(ids, arr, pr, out), logs=True)
        logs_equal = tlog == wt and dlog == wd
        ok = csv == wcsv and logs_equal and s["kv_words_mismatched"] == 0 and s["requests_verified"] == len(ids)
        bad += not ok
        print(json.dumps({"seed": seed, "model": kind, "bs": bs, "tp_rank": tp_rank, "requests": n_req, "rate": rate, "gpu_blocks": gpu_blocks, "pinned": pinned,
                          "layerkv": layerkv, "escalations": s["escalations"], "decode_iterations": s["decode_iterations"],
                          "d2h_jobs": ws["d2h_jobs"], "h2d_jobs": ws["h2d_jobs"], "csv_equal": csv == wcsv, "cli_logs_equal": logs_equal,
                          "kv_words_mismatched": s["kv_words_mismatched"], "s": round(time.perf_counter() - t0, 1)}),
              flush=True)
    print(json.dumps({"traces": a.n, "mismatched": bad}))
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
