"""Causal GQA prefill attention.

The reference has no attention arithmetic: the oracle is the
fp64-accumulated CPU restatement oracle/attn_ref.c:oracle_prefill_attn, which
is itself pinned here against an independent numpy softmax. The device kernel
(tcgen05, paper_2410_00428_b200/csrc/prefill_attn.cuh) must match the oracle
within 1e-3 relative (fp32 output; max-abs error per row normalised by the
row's max |o|), per the north star.
"""
import math

import numpy as np
import pytest

import oracle
from tests import _device_scenarios as sc

REL_TOL = 1e-3


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def _bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _numpy_causal(q, k, v, scale):
    T, hq, d = q.shape
    g = hq // k.shape[1]
    qf, kf, vf = _bits_to_f64(q), _bits_to_f64(k), _bits_to_f64(v)
    out = np.empty((T, hq, d))
    for h in range(hq):
        s = qf[:, h, :] @ kf[:, h // g, :].T * scale
        s[np.triu_indices(T, 1)] = -np.inf
        p = np.exp(s - s.max(axis=1, keepdims=True))
        out[:, h, :] = (p / p.sum(axis=1, keepdims=True)) @ vf[:, h // g, :]
    return out


def _inputs(T, hq, hkv, d, seed, qscale=1.0):
    rng = np.random.default_rng(seed)
    q = _bf16_bits(rng.uniform(-1, 1, (T, hq, d)).astype(np.float32) * qscale)
    k = _bf16_bits(rng.uniform(-1, 1, (T, hkv, d)).astype(np.float32))
    v = _bf16_bits(rng.uniform(-1, 1, (T, hkv, d)).astype(np.float32))
    return q, k, v


def _rel_err(got, want):
    return float(sc.rel_err_rows(got, want).max())


@pytest.mark.parametrize("T,hq,hkv", [(1, 2, 1), (37, 4, 2), (130, 8, 2)])
def test_oracle_prefill_matches_numpy(T, hq, hkv):
    q, k, v = _inputs(T, hq, hkv, 128, seed=T)
    scale = 1 / math.sqrt(128)
    got = oracle.restatement().prefill_attn(q, k, v, scale)
    assert _rel_err(got, _numpy_causal(q, k, v, scale)) < 1e-6


def test_oracle_decode_is_last_prefill_row():
    """Decode attention over T keys = the last row of causal prefill over T tokens."""
    q, k, v = _inputs(50, 4, 2, 128, seed=5)
    re = oracle.restatement()
    scale = 1 / math.sqrt(128)
    pre = re.prefill_attn(q, k, v, scale)
    dec = re.decode_attn(q[-1], k, v, scale)
    assert _rel_err(dec, pre[-1]) < 1e-6


def _device(group, hkv=2):
    model = sc.gqa_model(L=2, hkv=hkv, group=group)
    return sc.make(model, gpu=64, cpu=64)


def _run_device(dev, q, k, v, scale, out_dtype):
    import torch
    from paper_2410_00428_b200.device import DTYPE_F32
    T, hq, d = q.shape
    tq = torch.from_numpy(q.view(np.int16)).view(torch.bfloat16).cuda()
    tk = torch.from_numpy(k.view(np.int16)).view(torch.bfloat16).cuda()
    tv = torch.from_numpy(v.view(np.int16)).view(torch.bfloat16).cuda()
    out = torch.empty((T, hq, d), dtype=torch.float32 if out_dtype == DTYPE_F32 else torch.bfloat16, device="cuda")
    dev.prefill_attention(tq, tk, tv, out, T, scale, out_dtype)
    dev.synchronize()
    return out.float().cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("group", [1, 2, 4, 8])
@pytest.mark.parametrize("T", [1, 100, 128, 129, 257, 385, 640, 1000])
def test_prefill_attention_parity(group, T):
    """Odd and even query-tile counts (a last CTA without its second tile),
    partial last tiles, every GQA group size."""
    from paper_2410_00428_b200.device import DTYPE_F32
    kv, dev = _device(group)
    q, k, v = _inputs(T, 2 * group, 2, 128, seed=1000 + T)
    scale = 1 / math.sqrt(128)
    got = _run_device(dev, q, k, v, scale, DTYPE_F32)
    want = oracle.restatement().prefill_attn(q, k, v, scale)
    err = _rel_err(got, want)
    assert err <= REL_TOL, f"prefill attention rel err {err:.3e}"
    dev.close()


@pytest.mark.gpu
def test_prefill_attention_sharp_softmax_rescales():
    """Scores spread over >> 2^8 in the log2 domain, with the max arriving in
    late tiles: exercises the lazy O rescale in TMEM."""
    from paper_2410_00428_b200.device import DTYPE_F32
    kv, dev = _device(4)
    T = 640
    q, k, v = _inputs(T, 8, 2, 128, seed=7, qscale=24.0)
    # grow the key norms with position so later tiles keep raising the row max
    kf = _bits_to_f64(k) * (1.0 + np.arange(T)[:, None, None] / 64.0)
    k = _bf16_bits(kf.astype(np.float32))
    scale = 1 / math.sqrt(128)
    got = _run_device(dev, q, k, v, scale, DTYPE_F32)
    want = oracle.restatement().prefill_attn(q, k, v, scale)
    assert _rel_err(got, want) <= REL_TOL
    dev.close()


@pytest.mark.gpu
def test_prefill_attention_bf16_output():
    from paper_2410_00428_b200.device import DTYPE_BF16
    kv, dev = _device(4)
    q, k, v = _inputs(300, 8, 2, 128, seed=3)
    scale = 1 / math.sqrt(128)
    got = _run_device(dev, q, k, v, scale, DTYPE_BF16)
    want = oracle.restatement().prefill_attn(q, k, v, scale)
    assert _rel_err(got, want) <= 8e-3  # bf16 storage of the output (2^-8 rounding)
    dev.close()
