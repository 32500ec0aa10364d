"""Shared pieces of the full-shape sampled parity checks (one GPU:
tests/test_gpu_fullshape.py; EP over NVLink: tests/mp_fullshape_check.py).

Parity is checked on samples whose oracle cost does not grow with the rest of
the batch (SURVEY.md §8c row sampling):
  - router logits on the sampled tokens (rel L2 <= 1e-4); the top-k choice and
    the gates of EVERY token bit-consistent with the GPU logits; the routing
    maps of every token (and every rank) bit-exact against the C oracle;
  - y, dx (incl. the router term) and dgates of the sampled tokens;
  - sampled intermediate columns j of every expert's dW1 (rows j and f+j) and
    dW2 (column j) over ALL tokens: column j needs only x.w1[j], x.w1[f+j] and
    dy.w2[:, j] per row (oracle/moe_oracle.c: orc_moe_wgrad_cols_bf16);
  - dW_r over all tokens from the GPU dgates (checked on the samples) through
    the softmax-over-selected backward.
Tolerances (relative L2 per tensor against the binary64 oracle on the same
bf16-valued inputs): bf16 path 1e-2, FP8 communication 5e-2 (dgates 7.5e-2, see
FP8_TOL_KEYS), and 1e-2 for y and dgates against the FP8-emulating reference
(fp8_emulated_rows).
"""
import os

import numpy as np
import torch

# FP8 communication against the plain oracle: the E4M3 rounding of x (per token)
# and of the fc2 output rows (grouped-128) each leave <= 2^-4 relative per element,
# ~2^-4/sqrt(3) = 3.6% rms; y / dx / dW average several such errors (measured
# 4.6%, bound 5e-2), a dgate is one dot product carrying both (sqrt(2) x 3.6% =
# 5.1% rms: bound 7.5e-2). Against the FP8-emulating reference (x and the fc2
# rows quantised exactly as the data path does) the same outputs are held to the
# bf16 path's 1e-2.
FP8_TOL_KEYS = {"dgates": 7.5e-2, "y_fp8emu": 1e-2, "dgates_fp8emu": 1e-2}

CONFIGS = {
    # BASELINE.json configs[1]: Mixtral-8x7B shape
    "cfg2_mixtral": dict(h=4096, f=14336, E=8, k=2, route="learned", comm="bf16", gate="before_fc2_in", tol=1e-2),
    # configs[2]: DeepSeek-V3 shape (fine-grained experts)
    "cfg3_deepseek": dict(h=7168, f=2048, E=256, k=8, route="learned", comm="bf16", gate="before_fc2_in", tol=1e-2),
    # configs[4]: Mixtral shape + FP8 communication + the reference's Zipf(1.2) routing
    "cfg5_fp8_zipf": dict(h=4096, f=14336, E=8, k=2, route="zipf", comm="fp8", gate="after_fc2_out", tol=5e-2,
                          tol_keys=FP8_TOL_KEYS),
    # configs[4] with the reference test's capacity factor 1.0 (test_routing.cpp:82-97):
    # group-capacity drops at EP > 1 (every rank one group, routing.cpp:113-131)
    "cfg5_fp8_zipf_cf1": dict(h=4096, f=14336, E=8, k=2, route="zipf", comm="fp8", gate="after_fc2_out", tol=5e-2,
                              cf=1.0, tol_keys=FP8_TOL_KEYS),
}
ZIPF_FIXTURE = "routing_cfg5_zipf_nodrop_n8.npz"


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def u16(t):
    return t.contiguous().cpu().view(torch.int16).numpy().view(np.uint16)


def _randn_bf16(shape, gen, scale):
    return (torch.randn(shape, generator=gen, device="cuda", dtype=torch.float32) * scale).bfloat16()


def make_inputs(c, T):
    """Full weights of all E experts and the whole batch, seeded on the GPU
    (identical on every rank of a box)."""
    h, f, E = c["h"], c["f"], c["E"]
    gw = torch.Generator(device="cuda").manual_seed(42)
    gx = torch.Generator(device="cuda").manual_seed(1234)
    w1 = _randn_bf16((E, 2 * f, h), gw, h ** -0.5)
    w2 = _randn_bf16((E, h, f), gw, f ** -0.5)
    wr = _randn_bf16((E, h), gw, h ** -0.5)
    x = _randn_bf16((T, h), gx, 0.5)
    dy = _randn_bf16((T, h), gx, 0.1)
    return w1, w2, wr, x, dy


def zipf_routing(golden_dir, T, k):
    """The reference's skewed routing (simulate_routing, Zipf s=1.2, seed 11;
    first T tokens) and fixed random gates."""
    g = np.load(os.path.join(golden_dir, ZIPF_FIXTURE))
    ex = g["experts"].astype(np.int32)[:T]
    rng = np.random.default_rng(0)
    gt = rng.random((T, k)).astype(np.float32) + 0.1
    gt /= gt.sum(1, keepdims=True)
    return ex, gt


def sample(T, f, n_tok=64, n_col=8, dropped=None):
    """Sampled tokens and intermediate columns. With capacity drops the tokens
    are drawn from the kept ones (a dropped token's outputs are exact zeros,
    checked over all of them by check_dropped_zero), so the numeric sample keeps
    its size whatever the drop rate."""
    rng = np.random.default_rng(7)
    if dropped is None:
        toks = np.unique(np.concatenate([[0, T - 1], rng.choice(T, n_tok, replace=False)]))
    else:
        pool = np.flatnonzero(np.asarray(dropped) == 0)
        toks = np.unique(np.concatenate([pool[:1], pool[-1:], rng.choice(pool, min(n_tok, pool.size), replace=False)]))
    cols = np.sort(rng.choice(f, n_col, replace=False))
    return toks, cols


def check_dropped_zero(dropped, y, dx, dgates):
    """Every dropped token (routing.cpp:113-131) contributes nothing: its y and
    dx rows and its dgates are exactly zero."""
    d = np.asarray(dropped) != 0
    assert not np.any(y[d]), "a dropped token has a non-zero output row"
    assert not np.any(dx[d]), "a dropped token has a non-zero dx row"
    assert not np.any(dgates[d]), "a dropped token has non-zero dgates"
    return int(d.sum())


def check_routing(P, c, ex, gt, dr, lg_all, toks, x, wr, n, Tr):
    """Router + top-k + every rank's scatter map; returns the logits error."""
    E, k = c["E"], c["k"]
    T = ex.shape[0]
    err = None
    if c["route"] == "learned":
        olg, _, _ = P.orc_router_topk(x.float().cpu().numpy()[toks], wr.float().cpu().numpy(), k)
        err = rel(lg_all[toks], olg)
        order = np.argsort(-lg_all, axis=1, kind="stable")[:, :k]
        assert (order == ex).all(), "top-k selection differs from the logits"
        sel = np.take_along_axis(lg_all, ex, 1).astype(np.float64)
        og = np.exp(sel - sel[:, :1])
        og /= og.sum(1, keepdims=True)
        assert np.abs(og - gt).max() < 1e-6, "gates differ from the softmax of the selected logits"
    src = (np.arange(T) // Tr).astype(np.int32)
    maps = [P.orc_build_scatter_map(ex, src, dr, E, n, r) for r in range(n)]
    return err, maps


def _bf16(a):
    """Round float32 values to bf16 (RNE), returned as float32."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def fp8_emulated_rows(P, ex, gt, toks, x, dy, w1, w2):
    """Forward y and the gate-after dgates of the sampled tokens with the FP8
    communication path emulated at its rounding points (gate after
    fc2, numerics.hpp:84-86): x quantised per token to E4M3 with the reference
    quantiser (numerics.cpp:113-160, the pinned C oracle) and dequantised in
    fp32 to bf16 as the dispatch does; fc1_out and fc2_in rounded to bf16;
    the fc2 output rows quantised grouped-128 and dequantised in fp32; y summed
    over the slots in fp32 and rounded to bf16; dgate = <dy, dequantised row>.
    The expert GEMMs are plain fp32 torch matmuls (TF32 off) on the GPU."""
    import torch
    tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        k = ex.shape[1]
        f = w1.shape[1] // 2
        xs = x[torch.from_numpy(np.asarray(toks)).to(x.device)].double().cpu().numpy()
        codes, sc = P.orc_quantize(xs, "per_token")
        xq = _bf16(codes.astype(np.float32) * sc.astype(np.float32)[:, None])
        rows = [(i, j, int(ex[t, j])) for i, t in enumerate(toks) for j in range(k)]
        out = np.zeros((len(toks), k, x.shape[1]), np.float32)
        for e in sorted({r[2] for r in rows}):
            sel = [(i, j) for i, j, ee in rows if ee == e]
            xe = torch.from_numpy(xq[[i for i, _ in sel]]).to(x.device)
            fc1 = _bf16((xe @ w1[e].float().T).cpu().numpy())
            a, b = fc1[:, :f], fc1[:, f:]
            h_in = _bf16(a * (b / (1.0 + np.exp(-b.astype(np.float64)))).astype(np.float32))
            fc2 = (torch.from_numpy(h_in).to(x.device) @ w2[e].float().T).cpu().numpy()
            c2, s2 = P.orc_quantize(fc2.astype(np.float64), "grouped", group_size=128)
            deq = c2.astype(np.float32) * np.repeat(s2.astype(np.float32).reshape(len(sel), -1), 128, axis=1)
            for q, (i, j) in enumerate(sel):
                out[i, j] = deq[q]
        y = np.zeros((len(toks), x.shape[1]), np.float32)
        for j in range(k):
            y = y + np.asarray(gt[toks, j], np.float32)[:, None] * out[:, j]
        dyt = dy[torch.from_numpy(np.asarray(toks)).to(dy.device)].double().cpu().numpy()
        dg = np.einsum("th,tjh->tj", dyt, out.astype(np.float64))
        return _bf16(y), dg
    finally:
        torch.backends.cuda.matmul.allow_tf32 = tf32


def dense_errors(P, c, ex, gt, dr, dg_all, toks, cols, x, dy, w1, w2, wr, y_tok, dx_tok, dw1_cols, dw2_cols, dwr):
    """y / dx / dgates of the sampled tokens, sampled wgrad columns of every
    expert, dW_r. dw1_cols [E, nc, 2, h] (rows j, f+j), dw2_cols [E, nc, h]."""
    E = c["E"]
    ga = c["gate"].startswith("after")
    learned = c["route"] == "learned"
    xu, dyu, w1u, w2u = u16(x), u16(dy), u16(w1), u16(w2)
    o = P.orc_moe_rows_bf16(xu, dyu, ex, gt, dr, w1u, w2u, u16(wr) if learned else None, toks, gate_after=ga)
    errs = dict(y=rel(y_tok, o["y"]), dgates=rel(dg_all[toks], o["dgates"]), dx=rel(dx_tok, o["dx"]))
    ow1, ow2 = P.orc_moe_wgrad_cols_bf16(xu, dyu, ex, gt, dr, w1u, w2u, cols, gate_after=ga)
    errs["dw1"] = rel(dw1_cols, ow1)
    errs["dw2"] = rel(dw2_cols, ow2)
    if learned:
        odwr = P.orc_router_wgrad_from_dgates(x.float().cpu().numpy(), ex, gt, dg_all, dr, E)
        errs["dwr"] = rel(dwr, odwr)
    if c["comm"] == "fp8" and ga:
        ey, edg = fp8_emulated_rows(P, ex, gt, toks, x, dy, w1, w2)
        errs["y_fp8emu"] = rel(y_tok, ey)
        errs["dgates_fp8emu"] = rel(dg_all[toks], edg)
    return errs


def tolerance(c, key):
    """Stated relative-L2 tolerance of output `key` for config c (module docstring)."""
    return c.get("tol_keys", {}).get(key, c["tol"])


def wgrad_cols(dw1, dw2, cols, f):
    """[E_local, nc, 2, h] and [E_local, nc, h] slices of the GPU weight grads."""
    ci = torch.from_numpy(cols).to(dw1.device)
    a = dw1.index_select(1, ci).float()
    b = dw1.index_select(1, ci + f).float()
    return torch.stack([a, b], 2), dw2.index_select(2, ci).float().transpose(1, 2).contiguous()
