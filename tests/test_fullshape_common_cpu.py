"""CPU checks of the full-shape parity helpers (tests/fullshape_common.py):
the bf16 rounding used by the FP8-emulating reference, the kept-token
sampling under capacity drops, and the stated tolerance table."""
import numpy as np
import torch

import fullshape_common as F


def test_bf16_rounding_matches_torch_rne():
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(200000) * np.exp(rng.uniform(-20, 20, 200000))).astype(np.float32)
    # exact halfway cases between two bf16 values (ties to even)
    u = rng.integers(0, 1 << 15, 5000, dtype=np.uint32) << 16 | 0x8000
    x = np.concatenate([x, u.view(np.float32)])
    x = x[np.isfinite(x)]
    want = torch.from_numpy(x).bfloat16().float().numpy()
    assert np.array_equal(F._bf16(x).view(np.uint32), want.view(np.uint32))


def test_sample_draws_kept_tokens_only():
    T = 16384
    dr = np.zeros(T, np.uint8)
    dr[np.random.default_rng(1).choice(T, T // 2, replace=False)] = 1
    toks, cols = F.sample(T, 14336, n_col=4, dropped=dr)
    assert len(toks) >= 64 and (dr[toks] == 0).all() and len(cols) == 4
    base, _ = F.sample(T, 14336, n_col=4)
    assert base[0] == 0 and base[-1] == T - 1


def test_tolerance_table():
    assert F.tolerance(F.CONFIGS["cfg2_mixtral"], "y") == 1e-2
    c = F.CONFIGS["cfg5_fp8_zipf_cf1"]
    assert F.tolerance(c, "y") == 5e-2 and F.tolerance(c, "dgates") == 7.5e-2
    assert F.tolerance(c, "y_fp8emu") == 1e-2 and F.tolerance(c, "dgates_fp8emu") == 1e-2
