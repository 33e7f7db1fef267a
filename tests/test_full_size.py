"""BASELINE.json configs at their real shapes, on the device path.

Config 1: LLaMA-2-7B (32 layers, 32 KV heads, d 128, block 16), one 1k-token
prefill with layer-wise offload (x = 0 / 16 / 32 retained layers), then 64
decode steps that append their tokens (f2) and re-fetch every CPU-resident
layer. Checked against the reference's own outputs (tests/golden, written by
the compiled reference): the block table's dump_table FNV hash after the
prefill and after 64 tokens and the final free counts; every KV byte of
every layer against the generator; attention of the first and last steps
against the fp32 restatement.

Config 4's per-GPU shard: Llama-3.1-70B GQA (80 layers, Hq 64 / Hkv 8) at
TP 8, rank 0 (one KV head, G = 8), 4k prompt with 40 retained layers (odd
layers kept, the reference placement), a few decode steps."""
from __future__ import annotations

import pytest

from paper_2410_00428_b200 import layersim as ls
from paper_2410_00428_b200.device import Device, DeviceConfig
from tests import _device_scenarios as sc
from tests.test_decode_append import _decode_step

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("x", [0, 16, 32])
def test_config1_full_size_against_reference(x, golden):
    g = golden["kv"][f"cfg1_x{x}"]
    model = ls.llama2_7b()
    kv = ls.KvManager(ls.BlockPools(200000, 800000, 16), model)
    dev = Device(kv, model, 16, DeviceConfig(gpu_slots=2304, host_slots=2304, arena_slots=160, max_requests=2,
                                             max_blocks=80, max_batch=1, staging_chunks=8, chunk_bytes=16 << 20))
    sc.prefill(kv, dev, 0, 1024, x)
    assert format(kv.dump_hash(), "016x") == g["after_prefill"]
    for step in range(64):
        _decode_step(kv, dev, [0], check=step in (0, 63))
    assert format(kv.dump_hash(), "016x") == g["after_64"]
    assert [(j.layer, j.bytes) for j in kv.plan_decode_fetch(0)] == [tuple(f) for f in g["fetch"]]
    assert (kv.gpu_blocks_free(), kv.cpu_blocks_free()) == (g["gpu_free"], g["cpu_free"])
    assert kv.request(0).cached_tokens == 1088
    assert dev.verify_request(0, 1088, sc.SEED) == 0
    dev.close()


def test_config4_tp8_shard_full_shape():
    model = ls.llama31_70b_gqa()
    kv = ls.KvManager(ls.BlockPools(2000000, 16000000, 16), model)
    prompt = 4096
    nblk = prompt // 16 + 2
    dev = Device(kv, model, 16, DeviceConfig(tp_rank=0, tp_size=8, gpu_slots=nblk * 40 + 64,
                                             host_slots=nblk * 40 + 64, arena_slots=nblk + 8, max_requests=2,
                                             max_blocks=nblk + 2, max_batch=1, staging_chunks=8,
                                             chunk_bytes=16 << 20))
    assert dev.kv_heads_local == 1 and dev.q_heads_local == 8
    sc.prefill(kv, dev, 0, prompt, 40)
    r = kv.request(0)
    assert [l for l in range(80) if r.layer_residency[l] == ls.LOC_GPU] == list(range(1, 80, 2))
    for step in range(3):
        _decode_step(kv, dev, [0], check=step == 2)
    assert dev.verify_request(0, prompt + 3, sc.SEED) == 0
    dev.close()
