"""Per-token E4M3 quantiser vs the reference's quantize (golden + oracle)."""
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_quantize_per_token_bit_exact():
    from paper_2505_11432_b200 import ops
    import pyoracle as P
    g = np.load(os.path.join(GOLDEN, "numerics.npz"))
    x = g["qx"].astype(np.float32)  # fp32-representable inputs
    codes, scales = ops.quantize_e4m3_rows(torch.from_numpy(x).cuda())
    want_codes, want_scales = P.orc_quantize(x.astype(np.float64), "per_token", "fp8_e4m3")
    got = torch.from_numpy(codes.cpu().numpy()).view(torch.float8_e4m3fn).float().numpy().astype(np.float64)
    assert (got == want_codes).all()
    np.testing.assert_array_equal(scales.cpu().numpy(), want_scales.astype(np.float32))
