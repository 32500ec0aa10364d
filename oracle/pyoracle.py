"""ctypes bindings for the CPU oracle (liboracle.so) and the reference build
(_ref/libmoeplan_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / reference arm, never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoeplan_ref.so")

_i64 = C.c_int64
_p = C.c_void_p


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def build(quiet: bool = True) -> None:
    """Compile the oracle (and _ref when /root/reference is present)."""
    import subprocess

    subprocess.run(["make", "-C", HERE, "all"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_orc = None
_ref = None


def oracle_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _orc = C.CDLL(ORACLE_SO)
        _orc.orc_round_to.restype = C.c_double
        _orc.orc_round_to.argtypes = [C.c_int, C.c_double]
        _orc.orc_build_scatter_map.restype = _i64
        _orc.orc_sort_tokens_for_tiles.restype = _i64
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        _ref = C.CDLL(REF_SO)
        _ref.ref_build_scatter_map.restype = _i64
        _ref.ref_sort_tokens_for_tiles.restype = _i64
    return _ref


# ----------------------------------------------------------------------------
# reference (oracle/_ref) wrappers
# ----------------------------------------------------------------------------
MODES = {"uniform": 0, "random": 1, "skewed": 2}


def ref_simulate_routing(T, E, k, mode="random", seed=0, zipf_s=1.0, cf=1e9, n_groups=1):
    lib = ref_lib()
    ex = np.zeros(T * k, np.int32)
    src = np.zeros(T, np.int32)
    dr = np.zeros(T, np.uint8)
    st = lib.ref_simulate_routing(_i64(T), _i64(E), _i64(k), C.c_int(MODES[mode]),
                                  C.c_uint64(seed), C.c_double(zipf_s), C.c_double(cf),
                                  _i64(n_groups), _p(_ptr(ex)), _p(_ptr(src)), _p(_ptr(dr)))
    if st != 0:
        raise ValueError(f"simulate_routing failed ({st})")
    return ex.reshape(T, k), src, dr


def ref_build_scatter_map(experts, src, dropped, E, n, my_rank, n_groups=None):
    lib = ref_lib()
    experts = np.ascontiguousarray(experts, np.int32)
    T, k = experts.shape
    src = np.ascontiguousarray(src, np.int32)
    dropped = np.ascontiguousarray(dropped, np.uint8)
    cap = max(T * k, 1)
    rmi, rmo, inv = (np.zeros(cap, np.int64) for _ in range(3))
    cnt = np.zeros(E, np.int64)
    oe, osr = np.zeros(cap, np.int32), np.zeros(cap, np.int32)
    rows = lib.ref_build_scatter_map(_i64(T), _i64(E), _i64(k), _i64(n_groups or n),
                                     _p(_ptr(experts)), _p(_ptr(src)), _p(_ptr(dropped)),
                                     _i64(n), _i64(my_rank), _p(_ptr(rmi)), _p(_ptr(rmo)),
                                     _p(_ptr(inv)), _p(_ptr(cnt)), _p(_ptr(oe)), _p(_ptr(osr)))
    if rows < 0:
        raise ValueError(f"build_scatter_map failed ({rows})")
    return dict(rows=int(rows), row_map_in=rmi[:rows], row_map_out=rmo[:rows],
                inverse_map=inv[:rows], per_expert_counts=cnt, out_expert=oe[:rows],
                out_source_rank=osr[:rows])


def ref_sort_tokens_for_tiles(experts, src, dropped, E, n, my_rank, tile_rows, n_groups=None):
    lib = ref_lib()
    experts = np.ascontiguousarray(experts, np.int32)
    T, k = experts.shape
    src = np.ascontiguousarray(src, np.int32)
    dropped = np.ascontiguousarray(dropped, np.uint8)
    cap = max(T * k, 1)
    te = np.zeros(cap, np.int32)
    tb, tend = np.zeros(cap, np.int64), np.zeros(cap, np.int64)
    tm = np.zeros(cap, np.uint64)
    lo, hi = np.zeros(cap, np.int32), np.zeros(cap, np.int32)
    nt = lib.ref_sort_tokens_for_tiles(_i64(T), _i64(E), _i64(k), _i64(n_groups or n),
                                       _p(_ptr(experts)), _p(_ptr(src)), _p(_ptr(dropped)),
                                       _i64(n), _i64(my_rank), _i64(tile_rows), _p(_ptr(te)),
                                       _p(_ptr(tb)), _p(_ptr(tend)), _p(_ptr(tm)), _p(_ptr(lo)),
                                       _p(_ptr(hi)))
    if nt < 0:
        raise ValueError(f"sort_tokens_for_tiles failed ({nt})")
    return dict(expert=te[:nt], begin=tb[:nt], end=tend[:nt], rank_mask=tm[:nt],
                rank_lo=lo[:nt], rank_hi=hi[:nt])


def ref_balance_metrics(experts, src, dropped, E, n):
    lib = ref_lib()
    experts = np.ascontiguousarray(experts, np.int32)
    T, k = experts.shape
    load = np.zeros(n, np.int64)
    loss, dr = C.c_double(), C.c_double()
    capv = C.c_int64()
    st = lib.ref_balance_metrics(_i64(T), _i64(E), _i64(k), _i64(n),
                                 _p(_ptr(experts)), _p(_ptr(np.ascontiguousarray(src, np.int32))),
                                 _p(_ptr(np.ascontiguousarray(dropped, np.uint8))), _i64(n),
                                 _p(_ptr(load)), C.byref(loss), C.byref(capv), C.byref(dr))
    if st != 0:
        raise ValueError(f"balance_metrics failed ({st})")
    return dict(per_group_load=load, loss=loss.value, capacity=capv.value, drop_rate=dr.value)


FORMATS = {"fp32": 0, "bf16": 1, "fp8_e4m3": 2}
GRANS = {"per_tensor": 0, "per_token": 1, "per_channel": 2, "grouped": 3}


def ref_round_to(fmt, x):
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty_like(x)
    ref_lib().ref_round_to(C.c_int(FORMATS[fmt]), _p(_ptr(x)), _i64(x.size), _p(_ptr(out)))
    return out


def _nblocks(rows, cols, gran, gs):
    return {0: 1, 1: rows, 2: cols, 3: rows * ((cols + gs - 1) // gs)}[gran] or 1


def ref_quantize(x, gran="per_token", fmt="fp8_e4m3", group_size=128):
    x = np.ascontiguousarray(x, np.float64)
    rows, cols = x.shape
    g = GRANS[gran]
    codes = np.zeros_like(x)
    scales = np.zeros(max(_nblocks(rows, cols, g, group_size), 1))
    nb = C.c_int64()
    st = ref_lib().ref_quantize(_p(_ptr(x)), _i64(rows), _i64(cols), C.c_int(g),
                                _i64(group_size), C.c_int(FORMATS[fmt]), _p(_ptr(codes)),
                                _p(_ptr(scales)), C.byref(nb))
    if st != 0:
        raise ValueError(f"quantize failed ({st})")
    return codes, scales[: nb.value]


def ref_emulate_reduce(vectors, kind="a2a_fp32"):
    v = np.ascontiguousarray(vectors, np.float64)
    out = np.zeros(v.shape[1])
    st = ref_lib().ref_emulate_reduce(_p(_ptr(v)), _i64(v.shape[0]), _i64(v.shape[1]),
                                      C.c_int(0 if kind == "ring_bf16" else 1), _p(_ptr(out)))
    if st != 0:
        raise ValueError(f"emulate_reduce failed ({st})")
    return out


# ----------------------------------------------------------------------------
# oracle (C restatement) wrappers
# ----------------------------------------------------------------------------
def orc_capacity_drop(experts, E, n_groups, cf):
    experts = np.ascontiguousarray(experts, np.int32)
    T, k = experts.shape
    dr = np.zeros(T, np.uint8)
    st = oracle_lib().orc_capacity_drop(_i64(T), _i64(E), _i64(k), _i64(n_groups),
                                        C.c_double(cf), _p(_ptr(experts)), _p(_ptr(dr)))
    if st != 0:
        raise ValueError("capacity_drop: invalid arguments")
    return dr


def orc_build_scatter_map(experts, src, dropped, E, n, my_rank):
    experts = np.ascontiguousarray(experts, np.int32)
    T, k = experts.shape
    cap = max(T * k, 1)
    rmi = np.zeros(cap, np.int64)
    cnt = np.zeros(E, np.int64)
    oe, osr = np.zeros(cap, np.int32), np.zeros(cap, np.int32)
    rows = oracle_lib().orc_build_scatter_map(
        _i64(T), _i64(E), _i64(k), _p(_ptr(experts)),
        _p(_ptr(np.ascontiguousarray(src, np.int32))),
        _p(_ptr(np.ascontiguousarray(dropped, np.uint8))), _i64(n), _i64(my_rank),
        _p(_ptr(rmi)), _p(_ptr(cnt)), _p(_ptr(oe)), _p(_ptr(osr)))
    if rows < 0:
        raise ValueError("build_scatter_map: invalid arguments")
    return dict(rows=int(rows), row_map_in=rmi[:rows], per_expert_counts=cnt,
                out_expert=oe[:rows], out_source_rank=osr[:rows])


def orc_sort_tokens_for_tiles(out_expert, out_source_rank, tile_rows):
    rows = len(out_expert)
    cap = max(rows, 1)
    te = np.zeros(cap, np.int32)
    tb, tend = np.zeros(cap, np.int64), np.zeros(cap, np.int64)
    tm = np.zeros(cap, np.uint64)
    nt = oracle_lib().orc_sort_tokens_for_tiles(
        _i64(rows), _p(_ptr(np.ascontiguousarray(out_expert, np.int32))),
        _p(_ptr(np.ascontiguousarray(out_source_rank, np.int32))), _i64(tile_rows),
        _p(_ptr(te)), _p(_ptr(tb)), _p(_ptr(tend)), _p(_ptr(tm)))
    return dict(expert=te[:nt], begin=tb[:nt], end=tend[:nt], rank_mask=tm[:nt])


def orc_balance_metrics(experts, dropped, E, n):
    experts = np.ascontiguousarray(experts, np.int32)
    T, k = experts.shape
    load = np.zeros(n, np.int64)
    loss, dr = C.c_double(), C.c_double()
    capv = C.c_int64()
    oracle_lib().orc_balance_metrics(_i64(T), _i64(E), _i64(k), _p(_ptr(experts)),
                                     _p(_ptr(np.ascontiguousarray(dropped, np.uint8))), _i64(n),
                                     _p(_ptr(load)), C.byref(loss), C.byref(capv), C.byref(dr))
    return dict(per_group_load=load, loss=loss.value, capacity=capv.value, drop_rate=dr.value)


def orc_round_to(fmt, x):
    f = FORMATS[fmt]
    lib = oracle_lib()
    x = np.asarray(x, np.float64)
    return np.array([lib.orc_round_to(f, float(v)) for v in x.ravel()]).reshape(x.shape)


def orc_quantize(x, gran="per_token", fmt="fp8_e4m3", group_size=128):
    x = np.ascontiguousarray(x, np.float64)
    rows, cols = x.shape
    g = GRANS[gran]
    codes = np.zeros_like(x)
    scales = np.zeros(max(_nblocks(rows, cols, g, group_size), 1))
    nb = C.c_int64()
    oracle_lib().orc_quantize(_p(_ptr(x)), _i64(rows), _i64(cols), C.c_int(g), _i64(group_size),
                              C.c_int(FORMATS[fmt]), _p(_ptr(codes)), _p(_ptr(scales)),
                              C.byref(nb))
    return codes, scales[: nb.value]


def orc_emulate_reduce(vectors, kind="a2a_fp32"):
    v = np.ascontiguousarray(vectors, np.float64)
    out = np.zeros(v.shape[1])
    oracle_lib().orc_emulate_reduce(_p(_ptr(v)), _i64(v.shape[0]), _i64(v.shape[1]),
                                    C.c_int(0 if kind == "ring_bf16" else 1), _p(_ptr(out)))
    return out


def orc_router_topk(x, wr, k):
    x = np.ascontiguousarray(x, np.float32)
    wr = np.ascontiguousarray(wr, np.float32)
    T, h = x.shape
    E = wr.shape[0]
    logits = np.zeros((T, E), np.float32)
    ex = np.zeros((T, k), np.int32)
    g = np.zeros((T, k), np.float32)
    oracle_lib().orc_router_topk(_p(_ptr(x)), _p(_ptr(wr)), _i64(T), _i64(h), _i64(E), _i64(k),
                                 _p(_ptr(logits)), _p(_ptr(ex)), _p(_ptr(g)))
    return logits, ex, g


def orc_moe_forward(x, experts, gates, dropped, w1, w2, tokens=None, gate_after=False):
    x = np.ascontiguousarray(x, np.float32)
    T, h = x.shape
    E, f2, _ = w1.shape
    f = f2 // 2
    k = experts.shape[1]
    tokens = np.arange(T, dtype=np.int64) if tokens is None else np.ascontiguousarray(tokens, np.int64)
    y = np.zeros((len(tokens), h), np.float32)
    oracle_lib().orc_moe_forward(
        _p(_ptr(x)), _p(_ptr(np.ascontiguousarray(experts, np.int32))),
        _p(_ptr(np.ascontiguousarray(gates, np.float32))),
        _p(_ptr(np.ascontiguousarray(dropped, np.uint8))),
        _p(_ptr(np.ascontiguousarray(w1, np.float32))), _p(_ptr(np.ascontiguousarray(w2, np.float32))),
        _i64(h), _i64(f), _i64(k), C.c_int(int(gate_after)), _p(_ptr(tokens)), _i64(len(tokens)),
        _p(_ptr(y)))
    return y


def orc_moe_backward(x, dy, experts, gates, logits, dropped, w1, w2, wr, tokens=None,
                     gate_after=False, weight_grads=True, out=None):
    """out: optional preallocated (dw1, dw2, dwr) fp32 buffers, zeroed here and
    accumulated into (saves the per-call allocation of weight-sized arrays)."""
    x = np.ascontiguousarray(x, np.float32)
    T, h = x.shape
    E, f2, _ = w1.shape
    f = f2 // 2
    k = experts.shape[1]
    tokens = np.arange(T, dtype=np.int64) if tokens is None else np.ascontiguousarray(tokens, np.int64)
    nt = len(tokens)
    dx = np.zeros((nt, h), np.float32)
    dg = np.zeros((nt, k), np.float32)
    if weight_grads and out is not None:
        dw1, dw2, dwr = out
        for a in out:
            a.fill(0.0)
    else:
        dw1 = np.zeros_like(w1, dtype=np.float32) if weight_grads else None
        dw2 = np.zeros_like(w2, dtype=np.float32) if weight_grads else None
        dwr = np.zeros((E, h), np.float32) if weight_grads else None
    nul = lambda a: _p(None) if a is None else _p(_ptr(a))  # noqa: E731
    oracle_lib().orc_moe_backward(
        _p(_ptr(x)), _p(_ptr(np.ascontiguousarray(dy, np.float32))),
        _p(_ptr(np.ascontiguousarray(experts, np.int32))),
        _p(_ptr(np.ascontiguousarray(gates, np.float32))),
        _p(_ptr(np.ascontiguousarray(logits, np.float32))),
        _p(_ptr(np.ascontiguousarray(dropped, np.uint8))),
        _p(_ptr(np.ascontiguousarray(w1, np.float32))), _p(_ptr(np.ascontiguousarray(w2, np.float32))),
        _p(_ptr(np.ascontiguousarray(wr, np.float32))), _i64(h), _i64(f), _i64(E), _i64(k),
        C.c_int(int(gate_after)), _p(_ptr(tokens)), _i64(nt), _p(_ptr(dx)), _p(_ptr(dg)),
        nul(dw1), nul(dw2), nul(dwr))
    return dict(dx=dx, dgates=dg, dw1=dw1, dw2=dw2, dwr=dwr)


# ----------------------------------------------------------------------------
# full-shape sampled parity (bf16 inputs, binary64 accumulation)
# ----------------------------------------------------------------------------
def _u16(a):
    """bf16 torch tensor / uint16 numpy array -> contiguous uint16 numpy."""
    if hasattr(a, "view") and hasattr(a, "dtype") and str(a.dtype) == "torch.bfloat16":
        import torch
        return a.contiguous().cpu().view(torch.int16).numpy().view(np.uint16)
    return np.ascontiguousarray(a, np.uint16)


def orc_moe_rows_bf16(x, dy, experts, gates, dropped, w1, w2, wr, tokens, gate_after=False):
    """y, dx, dgates of the sampled tokens. x/dy/w1/w2/wr are bf16 (torch) or
    their uint16 bit patterns; dy or wr may be None."""
    x, w1, w2 = _u16(x), _u16(w1), _u16(w2)
    dy = None if dy is None else _u16(dy)
    wr = None if wr is None else _u16(wr)
    T, h = x.shape
    E, f2, _ = w1.shape
    f = f2 // 2
    experts = np.ascontiguousarray(experts, np.int32)
    k = experts.shape[1]
    tokens = np.ascontiguousarray(tokens, np.int64)
    nt = len(tokens)
    y = np.zeros((nt, h), np.float32)
    dx = np.zeros((nt, h), np.float32)
    dg = np.zeros((nt, k), np.float32)
    nul = lambda a: _p(None) if a is None else _p(_ptr(a))  # noqa: E731
    oracle_lib().orc_moe_rows_bf16(
        _p(_ptr(x)), nul(dy), _p(_ptr(experts)), _p(_ptr(np.ascontiguousarray(gates, np.float32))),
        _p(_ptr(np.ascontiguousarray(dropped, np.uint8))), _p(_ptr(w1)), _p(_ptr(w2)), nul(wr),
        _i64(h), _i64(f), _i64(E), _i64(k), C.c_int(int(gate_after)), _p(_ptr(tokens)), _i64(nt),
        _p(_ptr(y)), _p(_ptr(dx)), _p(_ptr(dg)))
    return dict(y=y, dx=dx, dgates=dg)


def orc_moe_wgrad_cols_bf16(x, dy, experts, gates, dropped, w1, w2, cols, gate_after=False):
    """Sampled intermediate columns j of dW1 (rows j and f+j) and dW2 (column j)
    over all tokens: returns dw1 [E, nc, 2, h] and dw2 [E, nc, h] (fp32)."""
    x, dy, w1, w2 = _u16(x), _u16(dy), _u16(w1), _u16(w2)
    T, h = x.shape
    E, f2, _ = w1.shape
    f = f2 // 2
    experts = np.ascontiguousarray(experts, np.int32)
    k = experts.shape[1]
    cols = np.ascontiguousarray(cols, np.int64)
    nc = len(cols)
    dw1 = np.zeros((E, nc, 2, h), np.float32)
    dw2 = np.zeros((E, nc, h), np.float32)
    oracle_lib().orc_moe_wgrad_cols_bf16(
        _p(_ptr(x)), _p(_ptr(dy)), _p(_ptr(experts)), _p(_ptr(np.ascontiguousarray(gates, np.float32))),
        _p(_ptr(np.ascontiguousarray(dropped, np.uint8))), _p(_ptr(w1)), _p(_ptr(w2)), _i64(T), _i64(h),
        _i64(f), _i64(E), _i64(k), C.c_int(int(gate_after)), _p(_ptr(cols)), _i64(nc), _p(_ptr(dw1)),
        _p(_ptr(dw2)))
    return dw1, dw2


def orc_router_wgrad_from_dgates(x, experts, gates, dgates, dropped, E):
    """dW_r[E, h] = dlogits^T x with dlogits from the softmax-over-selected
    backward (dl_e = g_e (dg_e - sum_j g_j dg_j)); x fp32 [T, h]."""
    x = np.asarray(x, np.float64)
    T, k = experts.shape
    g = gates.astype(np.float64)
    dg = dgates.astype(np.float64)
    sdg = (g * dg).sum(1, keepdims=True)
    dl = g * (dg - sdg)
    dl[dropped.astype(bool)] = 0.0
    D = np.zeros((T, E))
    np.add.at(D, (np.repeat(np.arange(T), k), experts.reshape(-1)), dl.reshape(-1))
    return D.T @ x


def ref_time_routing(experts, src, dropped, E, n, tile_rows=128, reps=3):
    """Reference build_scatter_map x n, sort_tokens_for_tiles x n and
    balance_metrics timed inside the reference library (value types built once
    outside the timed region); returns the three medians in ms."""
    experts = np.ascontiguousarray(experts, np.int32)
    T, k = experts.shape
    ms = np.zeros(3)
    st = ref_lib().ref_time_routing(_i64(T), _i64(E), _i64(k), _i64(n), _p(_ptr(experts)),
                                    _p(_ptr(np.ascontiguousarray(src, np.int32))),
                                    _p(_ptr(np.ascontiguousarray(dropped, np.uint8))), _i64(n), _i64(tile_rows),
                                    C.c_int(reps), _p(_ptr(ms)))
    if st != 0:
        raise ValueError(f"ref_time_routing failed ({st})")
    return ms


def ref_time_numerics(x, vectors, gran="per_token", fmt="fp8_e4m3", group_size=128, kind="a2a_fp32"):
    """Reference quantize and emulate_reduce timed inside the library (ms)."""
    x = np.ascontiguousarray(x, np.float64)
    v = np.ascontiguousarray(vectors, np.float64)
    ms = np.zeros(2)
    st = ref_lib().ref_time_numerics(_p(_ptr(x)), _i64(x.shape[0]), _i64(x.shape[1]), C.c_int(GRANS[gran]),
                                     _i64(group_size), C.c_int(FORMATS[fmt]), _p(_ptr(v)), _i64(v.shape[0]),
                                     _i64(v.shape[1]), C.c_int(0 if kind == "ring_bf16" else 1), _p(_ptr(ms)))
    if st != 0:
        raise ValueError(f"ref_time_numerics failed ({st})")
    return ms


# ----------------------------------------------------------------------------
# fp32 numpy/BLAS restatement of the dense layer (CPU baseline at full shape)
# ----------------------------------------------------------------------------
def np_router_topk(x, wr, k):
    """logits = x wr^T; top-k (ties -> lower expert id); softmax over the k."""
    logits = x @ wr.T
    ex = np.argsort(-logits, axis=1, kind="stable")[:, :k].astype(np.int32)
    sel = np.take_along_axis(logits, ex, 1).astype(np.float64)
    g = np.exp(sel - sel[:, :1])
    g /= g.sum(1, keepdims=True)
    return logits, ex, g.astype(np.float32)


def np_moe_fwd_bwd(x, dy, wr, w1, w2, k, experts=None, gates=None, dropped=None, out=None):
    """The same math as orc_moe_forward / orc_moe_backward (graph.cpp:288-296
    forward, :333-401 backward; SwiGLU a*silu(b), gate before fc2, softmax
    router backward), batched per expert with fp32 BLAS GEMMs. Returns y, dx,
    dgates, (dw1, dw2, dwr); `out` = optional preallocated (dw1, dw2, dwr)."""
    T, h = x.shape
    E, f2, _ = w1.shape
    f = f2 // 2
    if experts is None:
        logits, experts, gates = np_router_topk(x, wr, k)
    dropped = np.zeros(T, bool) if dropped is None else dropped.astype(bool)
    y = np.zeros((T, h), np.float32)
    dx = np.zeros((T, h), np.float32)
    dg = np.zeros((T, k), np.float32)
    if out is None:
        out = (np.empty_like(w1), np.empty_like(w2), np.empty((E, h), np.float32))
    dw1, dw2, dwr = out
    flat_e = experts.reshape(-1)
    keep = ~np.repeat(dropped, k)
    for e in range(E):
        idx = np.nonzero((flat_e == e) & keep)[0]
        if idx.size == 0:
            dw1[e] = 0.0
            dw2[e] = 0.0
            continue
        t_idx, s_idx = idx // k, idx % k
        g = gates[t_idx, s_idx][:, None]
        xe = x[t_idx]
        h1 = xe @ w1[e].T
        a, b = h1[:, :f], h1[:, f:]
        sb = 1.0 / (1.0 + np.exp(-b))
        silu = b * sb
        z = a * silu * g
        y[t_idx] += z @ w2[e].T
        dout = dy[t_idx]
        dz = dout @ w2[e]
        dw2[e] = dout.T @ z
        dg[t_idx, s_idx] = (dz * a * silu).sum(1)
        dh1 = np.concatenate([dz * g * silu, dz * g * a * (sb * (1.0 + b * (1.0 - sb)))], 1)
        dw1[e] = dh1.T @ xe
        dx[t_idx] += dh1 @ w1[e]
    sdg = (gates * dg).sum(1, keepdims=True)
    dl = gates * (dg - sdg)
    dl[dropped] = 0.0
    dlog = np.zeros((T, E), np.float32)
    np.put_along_axis(dlog, experts.astype(np.int64), dl, 1)
    dx += dlog @ wr
    dwr[...] = dlog.T @ x
    return y, dx, dg, (dw1, dw2, dwr)
