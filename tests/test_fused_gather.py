"""Fused all-gather of per-head decode outputs (include/lkv.h
lkv_device_gather_*): the split-merge kernel stores each finished row into
every rank's gather buffer and publishes a per-layer epoch flag.

Nothing here needs more than one GPU: the ranks are lkv_devices on cuda:0 —
two in one process (raw pointers), and two processes that open each other's
buffers through CUDA IPC, the exact path bench.py takes at N>1. The gathered
rows must equal the concatenation of every rank's own output, bit for bit,
over several iterations (layer parity and epochs wrap)."""
from __future__ import annotations

import math
import os

import pytest

pytestmark = pytest.mark.gpu

L, HKV, GROUP, D = 3, 8, 4, 128
PROMPTS = [(0, 130, 1), (1, 40, 1), (2, 300, 0)]


def _rank_device(rank, world):
    from tests import _device_scenarios as sc
    model = sc.gqa_model(L=L, hkv=HKV, group=GROUP)
    kv, dev = sc.make(model, tp_rank=rank, tp_size=world)
    for rid, prompt, x in PROMPTS:
        sc.prefill(kv, dev, rid, prompt, x)
    return kv, dev


def _iterate(devs, iters=2):
    """Per layer: every rank's decode_layer, then every rank's wait + copy of
    the gathered rows (the consume-before-next-but-one-layer rule)."""
    import torch
    from tests import _device_scenarios as sc
    ids = [p[0] for p in PROMPTS]
    n = len(ids)
    scale = 1.0 / math.sqrt(D)
    results = []
    for it in range(iters):
        streams = [dev.torch_stream("compute") for dev in devs]
        qs = [[sc.random_q(n, devs[0].q_heads_local, D, 7000 + 100 * it + 10 * l + r).to("cuda:0")
               for l in range(L)] for r in range(len(devs))]
        outs = [[torch.empty((n, dev.q_heads_local, D), dtype=torch.bfloat16, device="cuda:0") for _ in range(L)]
                for dev in devs]
        got = [[None] * L for _ in devs]
        torch.cuda.synchronize()
        for dev in devs:
            dev.decode_begin(ids)
        for l in range(L):
            for r, dev in enumerate(devs):
                dev.decode_layer(l, qs[r][l], outs[r][l], scale, stream=streams[r])
            for r, dev in enumerate(devs):
                dev.gather_wait(l, stream=streams[r])
                with torch.cuda.stream(streams[r]):
                    got[r][l] = dev.gathered(l)[:n].clone()
        for dev in devs:
            dev.decode_end()
            dev.synchronize()
        torch.cuda.synchronize()
        results.append((outs, got))
    return results


def test_fused_gather_same_process():
    import torch
    world = 2
    pairs = [_rank_device(r, world) for r in range(world)]
    devs = [d for _, d in pairs]
    bases = [d.gather_buffer() for d in devs]
    for d in devs:
        d.gather_connect(bases)
    for outs, got in _iterate(devs, iters=3):
        for l in range(L):
            want = torch.cat([outs[r][l] for r in range(world)], dim=1)
            for r in range(world):
                assert torch.equal(got[r][l], want), f"rank {r} layer {l}: gathered rows differ"
    for d in devs:
        d.close()


def _ipc_worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        _, dev = _rank_device(rank, world)
        handles = [None] * world
        dist.all_gather_object(handles, dev.gather_ipc_handle())
        dev.gather_connect_ipc(handles)
        dist.barrier()
        bad = []
        for it, (outs, got) in enumerate(_iterate([dev], iters=3)):
            for l in range(L):
                every = [None] * world
                dist.all_gather_object(every, outs[0][l].cpu())
                want = torch.cat(every, dim=1)
                if not torch.equal(got[0][l].cpu(), want):
                    bad.append((it, l))
        dist.barrier()
        dev.close()
        dist.destroy_process_group()
        q.put((rank, bad))
    except BaseException as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def test_fused_gather_ipc_two_processes():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: [] for r in range(world)}, res
