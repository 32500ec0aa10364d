"""CPU check of the E4M3 fast-path argument used by the layer's hot
quantisers (csrc/common.cuh: e4m3_block / e4m3_code).

The kernels compute q = x * fp32(1/scale) in fp32 and convert with one RNE
cvt, falling back to the binary64 division x / scale of the reference
(numerics.cpp:149-156) only when q lies within 2^-16 quanta of an E4M3
rounding midpoint. This test emulates that arithmetic exactly with numpy
float32 and torch's RNE float32 -> e4m3 conversion, and checks against the
oracle's binary64 round_to that every value NOT sent to the fallback gets
the reference code — on random inputs and on inputs packed against the
midpoints, with scales that are not powers of two.
"""
import numpy as np
import torch

import pyoracle as P


def _near_midpoint(q):
    a = np.abs(q).astype(np.float32)
    bits = a.view(np.uint32)
    e = (bits >> 23).astype(np.int64) - 127
    e = np.maximum(e, -6)
    t = a * np.exp2(-(e - 3)).astype(np.float32)          # exact power-of-two scaling
    return np.abs(t - np.floor(t) - np.float32(0.5)) < np.float32(2.0 ** -16)


def _fast_codes(x, amax):
    scale = np.where(amax > 0, amax.astype(np.float64) / 448.0, 1.0)
    inv = (1.0 / scale).astype(np.float32)
    q = (x.astype(np.float32) * inv).astype(np.float32)       # one fp32 rounding, as FMUL
    q_sat = np.clip(q, -448.0, 448.0).astype(np.float32)      # cvt.satfinite
    codes = torch.from_numpy(q_sat).to(torch.float8_e4m3fn).double().numpy()
    fallback = _near_midpoint(q) & (np.abs(q) < 464.0)
    return codes, fallback, scale


def _exact_codes(x, scale):
    return P.orc_round_to("fp8_e4m3", x.astype(np.float64) / scale)


def test_fast_path_agrees_with_binary64_off_the_midpoints():
    rng = np.random.default_rng(1)
    n = 60000
    amax = (rng.random(n) * 10.0 ** rng.uniform(-8, 4, n)).astype(np.float32)
    x = (amax * rng.uniform(-1, 1, n)).astype(np.float32)
    # half of the values packed within a few fp32 ulps of E4M3 midpoints
    scale = amax.astype(np.float64) / 448.0
    m = rng.integers(8, 16, n) + 0.5
    quantum = np.exp2(rng.integers(-9, 5, n).astype(np.float64))
    target = m * quantum * (1.0 + rng.integers(-64, 65, n) * 2.0 ** -24)
    sel = rng.random(n) < 0.5
    x[sel] = np.clip(target[sel] * scale[sel], -amax[sel], amax[sel]).astype(np.float32)
    codes, fallback, sc = _fast_codes(x, amax)
    want = _exact_codes(x, sc)
    ok = ~fallback
    assert ok.sum() > n // 3
    bad = ok & (codes != want)
    assert not bad.any(), (x[bad][:5], amax[bad][:5])
    # the fallback is the reference arithmetic itself
    assert fallback.sum() > 0


def test_fast_path_bf16_inputs_and_power_of_two_scales():
    """bf16 rows (the dispatch payload) incl. exact ties: amax = 448 * 2^j
    makes x / scale exact, so E4M3 midpoints occur as exact ties."""
    rng = np.random.default_rng(2)
    n = 40000
    x = torch.from_numpy(rng.standard_normal(n).astype(np.float32) * 3).bfloat16().float().numpy()
    amax = np.full(n, 448.0 * 2.0 ** -3, np.float32)
    ties = (rng.integers(8, 16, n) + 0.5) * 2.0 ** rng.integers(-9, 3, n).astype(np.float64) * 2.0 ** -3
    x[: n // 2] = np.clip(ties[: n // 2], 0, 56.0).astype(np.float32)
    codes, fallback, sc = _fast_codes(x, amax)
    want = _exact_codes(x, sc)
    assert not (~fallback & (codes != want)).any()
