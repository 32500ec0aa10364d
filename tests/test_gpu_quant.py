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


def _lib():
    import ctypes as C
    from paper_2505_11432_b200 import lib
    L = lib()
    L.moe_quantize_num_blocks.restype = C.c_int64
    L.moe_quantize_workspace_size.restype = C.c_size_t
    return L


def test_round_to_bit_exact_vs_reference_golden():
    import ctypes as C
    L = _lib()
    g = np.load(os.path.join(GOLDEN, "numerics.npz"))
    x = torch.from_numpy(g["x"]).cuda()
    for fid, name in ((0, "fp32"), (1, "bf16"), (2, "fp8_e4m3")):
        out = torch.empty_like(x)
        assert L.moe_round_to(fid, C.c_void_p(x.data_ptr()), C.c_int64(x.numel()), C.c_void_p(out.data_ptr()), None) == 0
        got, want = out.cpu().numpy(), g[f"round_{name}"]
        assert ((got == want) | (np.isnan(got) & np.isnan(want))).all(), name


def test_quantize_all_granularities_bit_exact_vs_reference_golden():
    import ctypes as C
    L = _lib()
    g = np.load(os.path.join(GOLDEN, "numerics.npz"))
    q = g["qx"]
    rows, cols = q.shape
    xd = torch.from_numpy(q).cuda()
    for gid, name in enumerate(("per_tensor", "per_token", "per_channel", "grouped")):
        nb = L.moe_quantize_num_blocks(C.c_int64(rows), C.c_int64(cols), gid, C.c_int64(128))
        codes = torch.empty_like(xd)
        scales = torch.empty(nb, dtype=torch.float64, device="cuda")
        ws = torch.empty(int(L.moe_quantize_workspace_size(C.c_int64(rows), C.c_int64(cols), gid, C.c_int64(128))),
                         dtype=torch.uint8, device="cuda")
        st = L.moe_quantize(C.c_void_p(xd.data_ptr()), C.c_int64(rows), C.c_int64(cols), gid, C.c_int64(128), 2,
                            C.c_void_p(codes.data_ptr()), C.c_void_p(scales.data_ptr()), C.c_void_p(ws.data_ptr()), None)
        assert st == 0
        assert (codes.cpu().numpy() == g[f"q_{name}_codes"]).all(), name
        assert (scales.cpu().numpy() == g[f"q_{name}_scales"]).all(), name


def test_emulate_reduce_bit_exact_vs_reference_golden():
    import ctypes as C
    L = _lib()
    g = np.load(os.path.join(GOLDEN, "numerics.npz"))
    v = torch.from_numpy(g["rv"]).cuda()
    for kid, name in ((0, "ring_bf16"), (1, "a2a_fp32")):
        out = torch.empty(v.shape[1], dtype=torch.float64, device="cuda")
        assert L.moe_emulate_reduce(C.c_void_p(v.data_ptr()), C.c_int64(v.shape[0]), C.c_int64(v.shape[1]), kid,
                                    C.c_void_p(out.data_ptr()), None) == 0
        assert (out.cpu().numpy() == g[f"reduce_{name}"]).all(), name


def test_reference_test_numerics_against_gpu_adapter():
    """The reference's own tests/test_numerics.cpp, compiled unmodified against
    the drop-in numerics adapter (round_to / quantize / emulate_reduce on the GPU)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "oracle", "_ref", "ref_test_numerics_on_gpu")
    if not os.path.exists(exe):
        pytest.skip("reference test binary not built (needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(p.stdout[-3000:])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
