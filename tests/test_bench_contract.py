"""bench.py keeps the driver's JSON contract, at N=1 and on the N>1 path
(torchrun, gloo control plane, fused all-gather over CUDA IPC). The N>1 check
puts both ranks on cuda:0 (LKV_BENCH_ONE_GPU=1): it exercises the code path,
not the numbers."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"}


def _last_json(out: str):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
def test_bench_single_gpu_contract():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3", "--batch", "2", "--ctx", "2048",
                        "--no-rows", "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    assert KEYS <= set(line)
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["host_link"]["kv_verified_mismatches"] == 0
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(line["roofline"])
    assert line["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_bench_two_ranks_fused_allgather_path():
    env = dict(os.environ, LKV_BENCH_ONE_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
                        "--steps", "2", "--warmup", "3", "--batch", "2", "--ctx", "2048", "--no-rows",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    assert line["n_gpus"] == 2 and line["config"]["allgather"].startswith("fused")
    assert line["host_link"]["kv_verified_mismatches"] == 0


def test_reference_arm_contract():
    """--impl reference: rank 0 prints the reference line (oracle CPU port
    here), with impl/cpu_baseline/e2e keys."""
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--batch", "1", "--ctx", "1024"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    if r.returncode != 0 and "oracle" in r.stderr and "not built" in r.stderr:
        pytest.skip("oracle not built")
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    assert line["impl"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["cores"] >= 1


def test_reference_arm_loads_no_product_code():
    """The reference arm neither imports the product package nor maps liblkv.so."""
    code = ("import runpy, sys\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', '--batch', '1',"
            " '--ctx', '512']\n"
            "runpy.run_path('bench.py', run_name='__main__')\n"
            "maps = open('/proc/self/maps').read()\n"
            "print('PRODUCT_MODULES', [m for m in sys.modules if m.startswith('paper_2410_00428_b200')])\n"
            "print('LIBLKV_MAPPED', 'liblkv.so' in maps, 'libref_layersim.so' in maps)\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "PRODUCT_MODULES []" in r.stdout and "LIBLKV_MAPPED False True" in r.stdout, r.stdout[-500:]
