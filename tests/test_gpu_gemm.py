"""tcgen05 grouped GEMM vs a torch fp32 reference of the same op."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


@pytest.mark.parametrize("rows_per_group,N,K,bn", [
    ([128], 256, 64, 256), ([128], 256, 512, 256), ([256, 128, 384], 512, 1024, 256),
    ([128, 0, 256], 256, 256, 256), ([128] * 4, 384, 320, 128), ([512, 640], 1024, 4096, 256),
    ([256, 384], 512, 8192, 256),   # K >= 8192, several groups: single-lane issue, static stride
    ([384], 512, 8192, 256),        # K >= 8192, one group: convergent issue, dynamic tiles
])
@pytest.mark.parametrize("cta_pair", [False, True])
def test_m_grouped_kmajor(rows_per_group, N, K, bn, cta_pair):
    from paper_2505_11432_b200 import ops
    # cta_pair: 128-row multiples, odd counts end in an M=128 pair tile; bn = 128
    # with pairs = 256 x 128 tiles (the attention AG-GEMM's wave-fit variant)
    torch.manual_seed(1)
    G = len(rows_per_group)
    rows = sum(rows_per_group)
    a = torch.randn(rows, K, device="cuda").bfloat16()
    b = torch.randn(G * N, K, device="cuda").bfloat16()
    gr = torch.tensor(rows_per_group, dtype=torch.int32, device="cuda")
    for dt in (torch.float32, torch.bfloat16):
        out = ops.grouped_gemm(a, b, gr, N=N, K=K, out_dtype=dt, bn=bn, cta_pair=cta_pair)
        off = 0
        for g, r in enumerate(rows_per_group):
            if r == 0:
                continue
            ref = a[off:off + r].float() @ b[g * N:(g + 1) * N].float().T
            assert _rel(out[off:off + r], ref) < (1e-5 if dt == torch.float32 else 5e-3), (g, dt)
            off += r


@pytest.mark.parametrize("rows_per_group,N,K", [([128], 256, 64), ([256, 128], 512, 768), ([512, 384], 256, 512),
                                                 ([384, 256], 256, 8192)])
@pytest.mark.parametrize("cta_pair", [False, True])
def test_m_grouped_b_mnmajor(rows_per_group, N, K, cta_pair):
    from paper_2505_11432_b200 import ops
    torch.manual_seed(2)
    G = len(rows_per_group)
    rows = sum(rows_per_group)
    a = torch.randn(rows, K, device="cuda").bfloat16()
    b = torch.randn(G * K, N, device="cuda").bfloat16()   # per group [K, N]
    gr = torch.tensor(rows_per_group, dtype=torch.int32, device="cuda")
    out = ops.grouped_gemm(a, b, gr, N=N, K=K, b_mn_major=True, out_dtype=torch.float32, cta_pair=cta_pair)
    off = 0
    for g, r in enumerate(rows_per_group):
        ref = a[off:off + r].float() @ b[g * K:(g + 1) * K].float()
        assert _rel(out[off:off + r], ref) < 1e-5
        off += r


@pytest.mark.parametrize("rows_per_group,M,N", [([128], 256, 256), ([256, 0, 384], 512, 512)])
@pytest.mark.parametrize("cta_pair", [False, True])
def test_k_grouped_wgrad(rows_per_group, M, N, cta_pair):
    from paper_2505_11432_b200 import ops
    torch.manual_seed(3)
    G = len(rows_per_group)
    rows = sum(rows_per_group)
    a = torch.randn(rows, M, device="cuda").bfloat16()
    b = torch.randn(rows, N, device="cuda").bfloat16()
    gr = torch.tensor(rows_per_group, dtype=torch.int32, device="cuda")
    out = ops.grouped_gemm(a, b, gr, N=N, K=0, M=M, a_mn_major=True, b_mn_major=True,
                           k_grouped=True, out_dtype=torch.float32, cta_pair=cta_pair)
    off = 0
    for g, r in enumerate(rows_per_group):
        ref = a[off:off + r].float().T @ b[off:off + r].float()
        got = out[g * M:(g + 1) * M]
        if r == 0:
            assert got.abs().max().item() == 0.0
        else:
            assert _rel(got, ref) < 1e-5
        off += r
