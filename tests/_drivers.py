"""Shared drivers for the parity tests (test infrastructure).

* ``Rng``: restatement of the reference splitmix64 generator
  (proj/include/layersim/rng.hpp:12-65) so op streams match the reference's
  own tests seed for seed.
* ``fuzz_ops``: the random KvManager operation stream of
  proj/tests/test_kv_manager.cpp:265-322 (and variants), replayed through any
  library exposing the lkv C ABI; returns a trace of every observable result.
"""
from __future__ import annotations

import hashlib
import math

from paper_2410_00428_b200 import layersim as ls

MASK = (1 << 64) - 1


class Rng:
    def __init__(self, seed: int):
        self.state = seed & MASK

    @staticmethod
    def substream(seed: int, label: str, index: int = 0) -> "Rng":
        h = 1469598103934665603
        for ch in label.encode():
            h ^= ch
            h = (h * 1099511628211) & MASK
        r = Rng(seed ^ h)
        r.state = (r.state + 0x9E3779B97F4A7C15 * (index + 1)) & MASK
        r.next_u64()
        r.next_u64()
        return r

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform01(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def uniform_below(self, n: int) -> int:
        return self.next_u64() % n


def fuzz_ops(lib, seed=31, rounds=10, steps=300, gpu=256, cpu=512, model=None, max_prompt=64,
             check_every=1, record_tables=False, record_free=False, on_kv=None):
    """test_kv_manager.cpp:265-322 op mix, replayed through `lib`.

    Returns a list of per-op observations (all return values, free counts,
    dump hash), one list per round. record_free: also the two LIFO free
    stacks (kv_manager.hpp SlotPool). on_kv(kv) -> per-step callback or None
    (e.g. binds a Device and checks its mirror after every op)."""
    model = model or ls.tiny8()
    rng = Rng(seed)
    out = []
    for _ in range(rounds):
        kv = ls.KvManager(ls.BlockPools(gpu, cpu, 16), model, lib=lib)
        step_cb = on_kv(kv) if on_kv else None
        live, jobs, next_id = [], [], 0
        trace = []
        for step in range(steps):
            op = rng.uniform_below(5)
            obs = [op]
            if op == 0:
                x = rng.uniform_below(model.n_layers + 1)
                prompt = 1 + rng.uniform_below(max_prompt)
                ok = kv.allocate_prefill(next_id, prompt, x)
                obs += [x, prompt, ok]
                if ok:
                    live.append(next_id)
                next_id += 1
            elif op == 1 and live:
                rid = live[rng.uniform_below(len(live))]
                if kv.needs_append(rid):
                    obs += ["append", kv.append_decode_block(rid)]
                else:
                    kv.note_token(rid)
                    obs += ["note"]
            elif op == 2 and live:
                rid = live[rng.uniform_below(len(live))]
                mode = ls.HALF if rng.uniform_below(2) else ls.FULL
                before = (kv.offload_reclaim(rid, ls.HALF), kv.offload_reclaim(rid, ls.FULL),
                          kv.retained_layer_count(rid), kv.gpu_blocks_held(rid))
                job = kv.plan_offload(rid, mode)
                obs += [rid, mode, before, None if job is None else
                        (job.job_id, job.request_id, job.bytes, job.layer_count, job.gpu_blocks)]
                if job is not None and job.job_id >= 0:
                    jobs.append(job.job_id)
            elif op == 3 and jobs:
                j = jobs.pop()
                kv.complete_offload(j)
                obs += [j]
            elif op == 4 and live:
                pick = rng.uniform_below(len(live))
                f = kv.release(live[pick])
                obs += [f.gpu, f.cpu, f.deferred_gpu]
                del live[pick]
            kv.check_conservation()
            if step_cb:
                step_cb(step)
            if step % check_every == 0:
                obs += [kv.gpu_blocks_free(), kv.cpu_blocks_free(), format(kv.dump_hash(), "016x")]
                if record_free:
                    obs += [kv.free_stack(True), kv.free_stack(False)]
                for rid in live[:3]:
                    obs += [kv.gpu_row_cost(rid), kv.cpu_row_cost(rid),
                            [(j.layer, j.bytes) for j in kv.plan_decode_fetch(rid)]]
            trace.append(obs)
        for j in jobs:
            kv.complete_offload(j)
        for rid in live:
            kv.release(rid)
        if step_cb:
            step_cb(-1)
        trace.append(["final", kv.gpu_blocks_free(), kv.cpu_blocks_free()] +
                     ([kv.free_stack(True), kv.free_stack(False)] if record_free else []))
        out.append(trace)
    return out


def trace_digest(trace) -> str:
    return hashlib.sha256(repr(trace).encode()).hexdigest()


# ---------------------------------------------------------------- engine runs
ENGINE_FIELDS = [
    ("model", None), ("hw", None), ("cost", None),
]


def engine_cfg_struct(model: ls.ModelSpec, hw: ls.HardwareSpec, *, layerkv=True, slo=True, gpu_blocks, cpu_blocks,
                      tpb=16, seed=0, force_retained=-1, invariant_checks=False, max_batch_tokens=131072,
                      max_sim_time=86400.0, chunk_bytes=16.0 * 1024 * 1024, horizon=8, threshold=0.05,
                      accuracy=0.8, cost=None, ttft_slo=3.0, tpot_slo=0.2):
    import ctypes as C
    from paper_2410_00428_b200 import _abi

    class RefEngineCfg(C.Structure):
        _fields_ = [("model", _abi.ModelSpec), ("hw", _abi.HardwareSpec), ("cost", _abi.CostParams),
                    ("ttft_slo", C.c_double), ("tpot_slo", C.c_double), ("policy_layerkv", C.c_int32),
                    ("slo_scheduler", C.c_int32), ("gpu_blocks", C.c_int64), ("cpu_blocks", C.c_int64),
                    ("tokens_per_block", C.c_int32), ("horizon", C.c_int32), ("threshold_fraction", C.c_double),
                    ("predictor_accuracy", C.c_double), ("max_batch_tokens", C.c_int64),
                    ("max_sim_time", C.c_double), ("chunk_bytes", C.c_double), ("seed", C.c_uint64),
                    ("force_retained_layers", C.c_int32), ("invariant_checks", C.c_int32)]

    cost = cost or ls.CostParams()
    return RefEngineCfg(model.c(), hw.c(), cost.c(), ttft_slo, tpot_slo, int(layerkv), int(slo), gpu_blocks,
                        cpu_blocks, tpb, horizon, threshold, accuracy, max_batch_tokens, max_sim_time, chunk_bytes,
                        seed, force_retained, int(invariant_checks))


def generate_trace(lib, kind_sharegpt: bool, n: int, prompt: int, output: int, rate: float, seed: int):
    import ctypes as C
    ids = (C.c_int64 * n)()
    arr = (C.c_double * n)()
    p = (C.c_int32 * n)()
    o = (C.c_int32 * n)()
    st = lib.dll.ref_generate_trace(int(kind_sharegpt), n, prompt, output, rate, seed, ids, arr, p, o)
    assert st == 0, lib.dll.lkv_last_error()
    return list(ids), list(arr), list(p), list(o)


def run_engine(lib, cfg, trace):
    """Reference Engine::run through the shim; returns (summary dict, requests.csv)."""
    import ctypes as C

    class RefEngineOut(C.Structure):
        _fields_ = [("mean_ttft", C.c_double), ("p50_ttft", C.c_double), ("p99_ttft", C.c_double),
                    ("mean_tpot", C.c_double), ("throughput", C.c_double), ("makespan", C.c_double),
                    ("d2h_jobs", C.c_int64), ("h2d_jobs", C.c_int64), ("d2h_bytes", C.c_double),
                    ("h2d_bytes", C.c_double), ("completed", C.c_int32), ("n_rows", C.c_int32)]

    ids, arr, p, o = trace
    n = len(ids)
    out = RefEngineOut()
    ln = C.c_size_t()
    args = [C.byref(cfg), n, (C.c_int64 * n)(*ids), (C.c_double * n)(*arr), (C.c_int32 * n)(*p),
            (C.c_int32 * n)(*o), C.byref(out)]
    st = lib.dll.ref_engine_run(*args, None, 0, C.byref(ln))
    if st != 0:
        raise ls.SimulationError(lib.dll.lkv_last_error().decode())
    buf = C.create_string_buffer(ln.value + 1)
    lib.dll.ref_engine_run(*args, buf, ln.value + 1, C.byref(ln))
    summary = {k: getattr(out, k) for k, _ in out._fields_}
    return summary, buf.raw[:ln.value].decode()


def run_engine_log(lib, cfg, trace, which):
    """The reference run's transfer_log.csv (which="transfer") or
    decision_log.csv (which="decision"), Engine::transfer_log() /
    decision_log() in the CLI's format (tools/layersim_main.cpp:96-117),
    through the shim."""
    import ctypes as C
    ids, arr, p, o = trace
    n = len(ids)
    ln = C.c_size_t()
    args = [C.byref(cfg), n, (C.c_int64 * n)(*ids), (C.c_double * n)(*arr), (C.c_int32 * n)(*p),
            (C.c_int32 * n)(*o), 0 if which == "transfer" else 1]
    if lib.dll.ref_engine_log(*args, None, 0, C.byref(ln)) != 0:
        raise ls.SimulationError(lib.dll.lkv_last_error().decode())
    buf = C.create_string_buffer(ln.value + 1)
    lib.dll.ref_engine_log(*args, buf, ln.value + 1, C.byref(ln))
    return buf.raw[:ln.value].decode()


def isclose_rel(a, b, rel):
    return math.isclose(a, b, rel_tol=rel, abs_tol=0.0)
