"""Device-path scenarios shared by __graft_entry__.smoke() and the -m gpu tests.

Each scenario drives the product through the reference call sequence
(allocate_prefill -> per-layer prefill -> escalation plan/complete -> decode
iteration) and checks it against the oracle restatement: KV bytes bit-exact
with the generator wherever they live (GPU slots, pinned host frames, arena),
attention within 1e-3 relative (fp32 output) of the fp32 CPU restatement.
"""
from __future__ import annotations

import math

import numpy as np

from paper_2410_00428_b200 import layersim as ls
from paper_2410_00428_b200.device import DTYPE_BF16, DTYPE_F32, Device, DeviceConfig

SEED = 0x4C61796572
REL_TOL = 1e-3       # north star: attention within 1e-3 relative (fp32 accumulate)


def gqa_model(L=4, hkv=8, group=4, d=128):
    return ls.ModelSpec(L, hkv * group, hkv, d, hkv * group * d, 1.0e9, 2)


def make(model, bs=16, gpu=512, cpu=512, tp_rank=0, tp_size=1, depth=2, chunk_slots=3, max_blocks=64,
         max_batch=8, arena=None, pinned=0, device=0):
    """pinned > 0: tiered host memory (pageable homes for all `cpu` slots,
    `pinned` pinned frames)."""
    kv = ls.KvManager(ls.BlockPools(gpu, cpu, bs), model)
    slot_bytes = 2 * (model.n_kv_heads // tp_size) * bs * model.d_head * 2
    cfg = DeviceConfig(device=device, tp_rank=tp_rank, tp_size=tp_size, pipeline_depth=depth, gpu_slots=gpu,
                       host_slots=cpu, arena_slots=arena or gpu, max_requests=16, max_blocks=max_blocks,
                       max_batch=max_batch, staging_chunks=4, chunk_bytes=chunk_slots * slot_bytes,
                       pinned_frames=pinned)
    dev = Device(kv, model, bs, cfg)
    return kv, dev


def prefill(kv, dev, rid, prompt, x, seed=SEED):
    """allocate_prefill + per-layer K/V production + lkv_prefill_layer."""
    import torch
    assert kv.allocate_prefill(rid, prompt, x)
    L = dev.model.n_layers
    k = torch.empty((prompt, dev.kv_heads_local, dev.head_dim), dtype=torch.bfloat16,
                    device=f"cuda:{dev.cfg.device}")
    v = torch.empty_like(k)
    s = dev.torch_stream("compute")
    for layer in range(L):
        dev.fill_kv(k, v, prompt, 0, layer, seed, stream=s)
        dev.prefill_layer(rid, layer, k, v, prompt, stream=s)
    dev.synchronize()


def random_q(n, hq, d, gen_seed):
    import torch
    g = torch.Generator(device="cpu").manual_seed(gen_seed)
    return (torch.rand((n, hq, d), generator=g) * 2 - 1).to(torch.bfloat16)


def peaked_q(dev, layer, kv_lens, mode, seed=SEED, gen_seed=0):
    """Queries whose softmax is far from uniform, so the running-max paths run
    on their non-trivial branches (decode_gqa_tc.cuh lazy max, the split
    merge's rescale).

    mode "scaled": random q x 16 — scores of std ~5 (natural units) instead
    of ~0.3, so each 128-token tile has its own maximum.
    mode "rising": each query head is a weighted sum of the generator's keys
    at 4 anchor tokens (10%, 40%, 75%, 97% of the sequence) with weights
    2, 5, 8, 11: the scaled scores at the anchors are ~7.6, 19, 30 and 42
    against a background of std ~5, so the running maximum jumps by ~11
    (~16 in log2, past kLazyMax = 8) at tiles and chunks deep in the
    sequence, and the output is dominated by the last anchor's V.
    mode "extreme": weights 5, 20, 40, 60 — the last anchor's score (~227)
    stands ~160 (~230 in log2) above the background maximum of its tile's
    predecessors, past fp32's exponent range, so a kernel that stopped
    re-basing its running maximum would overflow."""
    import torch
    import oracle
    n = len(kv_lens)
    hq, hl, d = dev.q_heads_local, dev.kv_heads_local, dev.head_dim
    group = hq // hl
    coef = (5.0, 20.0, 40.0, 60.0) if mode == "extreme" else (2.0, 5.0, 8.0, 11.0)
    if mode == "scaled":
        return (random_q(n, hq, d, 2000 + layer + gen_seed).float() * 16).to(torch.bfloat16)
    re = oracle.restatement()
    g = np.random.default_rng(3000 + layer + gen_seed)
    q = np.zeros((n, hq, d), np.float32)
    for m, kv_len in enumerate(kv_lens):
        anchors = sorted({min(kv_len - 1, int(kv_len * f)) for f in (0.10, 0.40, 0.75, 0.97)})
        for i, t in enumerate(anchors):
            k, _ = re.fill_kv(1, t, layer, hl, dev.head0, d, seed)
            kf = (k.astype(np.uint32) << 16).view(np.float32)[0]  # [hl][d]
            c = coef[i + 4 - len(anchors)]
            q[m] += c * np.repeat(kf, group, axis=0)
        q[m] += g.uniform(-0.25, 0.25, size=(hq, d))
    return torch.from_numpy(q).to(torch.bfloat16)


def rel_err_rows(got, want):
    """Per-row relative error max|got - want| / max|want|, with a non-finite
    output row counted as +inf (NaN compares false: max(worst, nan) and
    nan > tol would otherwise let a NaN row pass)."""
    err = np.abs(got - want).max(axis=-1) / np.maximum(np.abs(want).max(axis=-1), 1e-30)
    return np.where(np.isfinite(err) & np.isfinite(got).all(axis=-1), err, np.inf)


def check_attention(dev, ids, kv_lens, seed=SEED, out_dtype=DTYPE_F32, layers=None, tol=None, q_mode=None):
    """One decode iteration over `ids`; every layer compared with the oracle.
    q_mode: None = U(-1, 1) queries; "scaled" / "rising" = peaked_q."""
    import torch
    import oracle
    re = oracle.restatement()
    n = len(ids)
    hq, d = dev.q_heads_local, dev.head_dim
    group = hq // dev.kv_heads_local
    scale = 1.0 / math.sqrt(d)
    L = dev.model.n_layers
    qs = [random_q(n, hq, d, 1000 + l) if q_mode is None else peaked_q(dev, l, kv_lens, q_mode, seed)
          for l in range(L)]
    outs = []
    dev.decode_begin(ids)
    for l in range(L):
        q = qs[l].to("cuda:0")
        out = torch.empty((n, hq, d), dtype=torch.float32 if out_dtype == DTYPE_F32 else torch.bfloat16,
                          device="cuda:0")
        dev.decode_layer(l, q, out, scale, out_dtype)
        outs.append(out)
    dev.decode_end()
    dev.synchronize()
    worst = 0.0
    limit = tol if tol is not None else (REL_TOL if out_dtype == DTYPE_F32 else 8e-3)
    where = []
    for l in (layers if layers is not None else range(L)):
        got = outs[l].float().cpu().numpy()
        q16 = qs[l].view(torch.int16).numpy().view(np.uint16)
        for m in range(n):
            want = re.decode_attn_gen(seed, l, kv_lens[m], dev.head0, dev.kv_heads_local, group, q16[m], scale)
            err = rel_err_rows(got[m], want)
            worst = max(worst, float(err.max()))
            if err.max() > limit:
                h = int(np.argmax(err))
                where.append(f"layer {l} member {m} (len {kv_lens[m]}) heads {np.nonzero(err > limit)[0].tolist()[:6]}"
                             f" got {got[m, h, :3]} want {want[h, :3]}")
    if where:  # diagnose: are the bytes themselves intact?
        bad = [dev.verify_request(rid, kv_lens[m], seed) for m, rid in enumerate(ids)]
        where.append(f"verify_request mismatches per member: {bad}")
    assert worst <= limit, f"attention rel err {worst:.3e} > {limit}: " + "; ".join(where[:10])
    return worst, outs


def smoke_scenario(verbose=False):
    """Prefill with layer-wise offload + escalation + one decode iteration."""
    model = gqa_model()
    kv, dev = make(model)
    prefill(kv, dev, 0, 100, 2)   # retained {1, 3}: scatter; {0, 2}: pack + D2H
    prefill(kv, dev, 1, 37, 4)    # all retained
    prefill(kv, dev, 2, 200, 0)   # all offloaded (multi-chunk D2H)
    job = kv.plan_offload(1, ls.HALF)  # escalation: gather + D2H of layers {0, 1}
    assert job is not None and job.job_id >= 0
    kv.complete_offload(job.job_id)    # waits for the copies, flips the table
    kv.check_conservation()
    for rid, n in ((0, 100), (1, 37), (2, 200)):
        bad = dev.verify_request(rid, n, SEED)
        assert bad == 0, f"request {rid}: {bad} KV elements differ from the generator"
    worst, _ = check_attention(dev, [0, 1, 2], [100, 37, 200])
    st = dev.decode_stats()
    pworst = check_prefill_attention(dev, 200)
    if verbose:
        print(f"smoke: bytes bit-exact; decode attention (tcgen05 GQA tile) max rel err {worst:.2e}; "
              f"prefill attention (tcgen05) max rel err {pworst:.2e}; "
              f"h2d {st.h2d_bytes_physical} B in {st.h2d_copies} copies; {st.attn_launches} attention launches")
    dev.close()
    return max(worst, pworst)


def check_prefill_attention(dev, T, seed=SEED):
    """Causal prefill attention of generator K/V (layer 0) through
    lkv_prefill_attention vs the fp64 oracle, fp32 output, 1e-3 relative."""
    import torch
    import oracle
    re = oracle.restatement()
    hq, hl, d = dev.q_heads_local, dev.kv_heads_local, dev.head_dim
    k = torch.empty((T, hl, d), dtype=torch.bfloat16, device="cuda:0")
    v = torch.empty_like(k)
    s = dev.torch_stream("compute")
    dev.fill_kv(k, v, T, 0, 0, seed, stream=s)
    q = random_q(T, hq, d, 4242).to("cuda:0")
    out = torch.empty((T, hq, d), dtype=torch.float32, device="cuda:0")
    torch.cuda.synchronize()
    dev.prefill_attention(q, k, v, out, T, 1.0 / math.sqrt(d), DTYPE_F32, stream=s)
    dev.synchronize()
    want = re.prefill_attn(q.cpu().view(torch.int16).numpy().view(np.uint16),
                           k.cpu().view(torch.int16).numpy().view(np.uint16),
                           v.cpu().view(torch.int16).numpy().view(np.uint16), 1.0 / math.sqrt(d))
    got = out.cpu().numpy()
    err = float(rel_err_rows(got, want).max())
    assert err <= REL_TOL, f"prefill attention rel err {err:.3e} > {REL_TOL}"
    return err
