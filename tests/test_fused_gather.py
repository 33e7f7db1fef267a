"""Fused all-gather of per-head decode outputs (include/lkv.h
lkv_device_gather_*): the split-merge kernel stores each finished row into
every rank's gather buffer and publishes a per-layer epoch flag.

Ranks are lkv_devices: two in one process (raw pointers) and two processes
that open each other's buffers through CUDA IPC (the exact path bench.py
takes at N>1), both on cuda:0 everywhere, and on distinct GPUs where the box
has two (peer stores over NVLink; skipped on one GPU). The gathered rows must
equal the concatenation of every rank's own output, bit for bit,
over several iterations (layer parity and epochs wrap)."""
from __future__ import annotations

import math
import os

import pytest

pytestmark = pytest.mark.gpu

L, HKV, GROUP, D = 3, 8, 4, 128
PROMPTS = [(0, 130, 1), (1, 40, 1), (2, 300, 0)]


def _rank_device(rank, world, device=0):
    from tests import _device_scenarios as sc
    model = sc.gqa_model(L=L, hkv=HKV, group=GROUP)
    kv, dev = sc.make(model, tp_rank=rank, tp_size=world, device=device)
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
        qs = [[sc.random_q(n, devs[0].q_heads_local, D, 7000 + 100 * it + 10 * l + r).to(f"cuda:{devs[r].cfg.device}")
               for l in range(L)] for r in range(len(devs))]
        outs = [[torch.empty((n, dev.q_heads_local, D), dtype=torch.bfloat16, device=f"cuda:{dev.cfg.device}")
                 for _ in range(L)] for dev in devs]
        got = [[None] * L for _ in devs]
        for dev in devs:
            torch.cuda.synchronize(dev.cfg.device)
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
        for dev in devs:
            torch.cuda.synchronize(dev.cfg.device)
        results.append((outs, got))
    return results


def _same_process(devices):
    import torch
    world = len(devices)
    pairs = [_rank_device(r, world, devices[r]) for r in range(world)]
    devs = [d for _, d in pairs]
    bases = [d.gather_buffer() for d in devs]
    for d in devs:
        d.gather_connect(bases)
    for r, d in enumerate(devs):  # peers on another GPU are reached over P2P, explicitly enabled
        assert d.placement()["gather_peers_p2p"] == sum(1 for x in devices if x != devices[r])
    for outs, got in _iterate(devs, iters=3):
        for l in range(L):
            for r in range(world):
                want = torch.cat([outs[p][l].to(f"cuda:{devices[r]}") for p in range(world)], dim=1)
                assert torch.equal(got[r][l], want), f"rank {r} layer {l}: gathered rows differ"
    for d in devs:
        d.close()


def test_fused_gather_same_process():
    _same_process([0, 0])


def test_fused_gather_two_devices_same_process():
    """Ranks on distinct GPUs in one process: the peer stores cross NVLink
    (peer access enabled by gather_connect). Skips on a one-GPU box."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    _same_process([0, 1])


def _ipc_worker(rank, world, port, q, distinct=False):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        device = rank if distinct else 0
        torch.cuda.set_device(device)
        _, dev = _rank_device(rank, world, device)
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


@pytest.mark.parametrize("distinct", [False, True])
def test_fused_gather_ipc_two_processes(distinct):
    """Two processes exchanging gather buffers through CUDA IPC (bench.py's
    N>1 path): both on cuda:0, and — on a box with two GPUs — one per GPU."""
    import socket

    import torch
    import torch.multiprocessing as mp
    if distinct and torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q, distinct)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: [] for r in range(world)}, res
