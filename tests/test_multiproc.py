"""World-size-2 gloo tests of the N>1 host logic (no GPU).

* Replicated bookkeeping: every rank drives its own KvManager through the same
  op stream; table hashes, free counts and fetch plans agree across ranks.
* KV-head sharding + the one collective: each rank computes attention for its
  head shard (oracle restatement on CPU, generator KV), all-gathers the
  per-head outputs, and the assembled result equals the unsharded attention.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import oracle
        from paper_2410_00428_b200 import layersim as ls
        from paper_2410_00428_b200 import tp
        from tests import _drivers as drv

        # ---- replicated table
        trace = drv.fuzz_ops(None, seed=5, rounds=2, steps=200, gpu=300, cpu=300)
        digest = drv.trace_digest(trace)
        obj = [None] * world
        dist.all_gather_object(obj, digest)
        assert len(set(obj)) == 1, "rank tables diverged"

        # ---- head shard + all-gather of outputs
        re = oracle.restatement()
        hkv, group, d, kv_len, seed = 8, 4, 128, 70, 77
        lo, hi = tp.kv_head_range(rank, world, hkv)
        qlo, qhi = tp.q_head_range(rank, world, hkv * group, hkv)
        rng = np.random.default_rng(3)
        q_full = (rng.standard_normal((hkv * group, d)).astype(np.float32))
        q16 = (q_full.view(np.uint32) >> 16).astype(np.uint16)
        scale = 1 / math.sqrt(d)
        local = re.decode_attn_gen(seed, 2, kv_len, lo, hi - lo, group, q16[qlo:qhi], scale)
        full = tp.all_gather_heads(dist, torch.from_numpy(local).unsqueeze(0))
        want = re.decode_attn_gen(seed, 2, kv_len, 0, hkv, group, q16, scale)
        assert torch.allclose(full[0], torch.from_numpy(want), rtol=0, atol=0), "assembled heads differ"
        assert tp.slot_bytes(16, 2 * 8 * 128 * 2, world) * world == 16 * 2 * 8 * 128 * 2
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))


def test_two_rank_gloo_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(results) == [(0, "ok"), (1, "ok")], results


def test_head_ranges_cover_and_partition():
    from paper_2410_00428_b200 import tp
    for hkv in (8, 32):
        for world in (1, 2, 4, 8):
            rs = [tp.kv_head_range(r, world, hkv) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == hkv
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    with pytest.raises(ValueError):
        tp.kv_head_range(0, 3, 8)
