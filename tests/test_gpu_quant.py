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


def _decode(codes_u8):
    return torch.from_numpy(codes_u8).view(torch.float8_e4m3fn).double().numpy()


def _stress_bf16_rows(rows, cols, seed):
    """bf16 rows with varied magnitudes: random, all-zero, tiny (amax below
    ~1.3e-36, where 1/scale overflows fp32), and power-of-two scales that make
    x/scale land exactly on E4M3 rounding midpoints (RNE ties)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((rows, cols)).astype(np.float32) * 10.0 ** rng.uniform(-3, 3, (rows, 1))
    x[1] = 0.0
    x[2] *= 1e-38
    ties = (rng.integers(8, 16, (8, cols)) + 0.5) * 2.0 ** rng.integers(-9, 3, (8, cols)).astype(np.float64)
    x[3:11] = np.clip(ties * np.sign(rng.standard_normal((8, cols))), -56.0, 56.0) / 8
    x[3:11, 0] = 56.0 / 8                     # amax = 448 * 2^-6: exact ties after scaling
    return torch.from_numpy(x).bfloat16()


@pytest.mark.parametrize("group", [0, 128])
def test_layer_dispatch_quantiser_bit_exact_vs_reference(group):
    """The quantiser the layer runs on its dispatch payloads (quantize_fast_kernel:
    per-token forward x, grouped-128 backward dy) against the reference's own
    quantize (oracle/_ref, numerics.cpp:113-160) on the same bf16 values."""
    import pyoracle as P
    from paper_2505_11432_b200 import ops
    xb = _stress_bf16_rows(64, 4096, 3)
    codes, scales = ops.quantize_e4m3_fast(xb.cuda(), group=group)
    x64 = xb.float().numpy().astype(np.float64)
    quant = P.ref_quantize if P.ref_available() else P.orc_quantize
    want_codes, want_scales = quant(x64, "per_token" if group == 0 else "grouped", "fp8_e4m3", 128)
    got = _decode(codes.cpu().numpy())
    assert (got == want_codes).all(), int((got != want_codes).sum())
    np.testing.assert_array_equal(scales.cpu().numpy().ravel(), want_scales.astype(np.float32))


@pytest.mark.parametrize("cta_pair", [False, True])
def test_combine_payload_epilogue_bit_exact_vs_reference(cta_pair):
    """EPI_SCATTER_FP8 (fc2 / fc1-dgrad FP8 combine payload): the grouped-128
    codes and scales it writes equal the reference quantize applied to the
    fp32 accumulators of the same GEMM (EPI_STORE_F32, same tiles)."""
    import pyoracle as P
    from paper_2505_11432_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(5)
    G, K, N = 3, 512, 1024
    rows = torch.tensor([256, 384, 128], dtype=torch.int32, device="cuda")
    R = int(rows.sum())
    a = (torch.randn(R, K, device="cuda", generator=g) * 0.5).bfloat16()
    b = (torch.randn(G * N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    acc = ops.grouped_gemm(a, b, rows, N=N, K=K, out_dtype=torch.float32, cta_pair=cta_pair)
    codes, scales = ops.grouped_gemm_e4m3(a, b, rows, N=N, K=K, cta_pair=cta_pair)
    torch.cuda.synchronize()
    quant = P.ref_quantize if P.ref_available() else P.orc_quantize
    want_codes, want_scales = quant(acc.cpu().numpy().astype(np.float64), "grouped", "fp8_e4m3", 128)
    got = _decode(codes.cpu().numpy())
    assert (got == want_codes).all(), int((got != want_codes).sum())
    np.testing.assert_array_equal(scales.cpu().numpy().ravel(), want_scales.astype(np.float32))
