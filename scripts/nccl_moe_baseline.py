"""Comparison baseline for the MoE layer (NOT the product): the standard
expert-parallel implementation with NCCL all-to-all dispatch / combine and
per-expert cuBLAS GEMMs through torch, forward + backward by hand (same math
and conventions as the fused layer: top-k softmax gates, SwiGLU a*silu(b),
gate before fc2). Used by bench.py to time the unfused NCCL path beside the
fused NVLink kernels on the same box, shapes and data.
"""
from __future__ import annotations

import torch
import torch.distributed as dist
import torch.nn.functional as F


class NcclMoEBaseline:
    def __init__(self, Tr, h, f, E, k, n, rank, w1, w2, wr):
        self.Tr, self.h, self.f, self.E, self.k, self.n, self.rank = Tr, h, f, E, k, n, rank
        self.el = E // n
        self.w1, self.w2, self.wr = w1, w2, wr  # [el, 2f, h], [el, h, f], [E, h]

    def _a2a(self, t, send_splits, recv_splits):
        if self.n == 1:
            return t
        out = t.new_empty((sum(recv_splits),) + tuple(t.shape[1:]))
        dist.all_to_all_single(out, t.contiguous(), recv_splits, send_splits)
        return out

    def step(self, x, dy):
        Tr, k, E, el, n = self.Tr, self.k, self.E, self.el, self.n
        # ---- forward ----
        logits = (x @ self.wr.T).float()
        topv, topi = logits.topk(k, dim=1)
        gates = torch.softmax(topv, dim=1)
        flat_e = topi.flatten()
        flat_t = torch.arange(Tr, device=x.device).repeat_interleave(k)
        order = torch.argsort(flat_e, stable=True)            # destination-rank-major (experts contiguous)
        dest = flat_e[order] // el
        send = torch.bincount(dest, minlength=n)
        recv = torch.empty_like(send)
        if n > 1:
            dist.all_to_all_single(recv, send)
        else:
            recv = send
        ss, rs = send.tolist(), recv.tolist()                  # host sync (split sizes)
        xin = self._a2a(x[flat_t[order]], ss, rs)
        e_in = self._a2a(flat_e[order].to(torch.int32), ss, rs)
        g_in = self._a2a(gates.flatten()[order], ss, rs)
        perm = torch.argsort(e_in, stable=True)
        xs, es, gs = xin[perm], e_in[perm], g_in[perm]
        counts = torch.bincount(es.long() - self.rank * el, minlength=el).tolist()
        outs, saved = [], []
        off = 0
        for j in range(el):
            c = counts[j]
            xe = xs[off:off + c]
            h1 = xe @ self.w1[j].T
            a, b = h1[:, :self.f], h1[:, self.f:]
            z = a * F.silu(b) * gs[off:off + c, None].to(a.dtype)
            outs.append(z @ self.w2[j].T)
            saved.append((xe, a, b, z))
            off += c
        out = torch.cat(outs) if outs else xs.new_zeros(0, self.h)
        back = torch.empty_like(out)
        back[perm] = out
        ret = self._a2a(back, rs, ss)
        y = torch.zeros(Tr, self.h, dtype=torch.float32, device=x.device)
        y.index_add_(0, flat_t[order], ret.float())
        y = y.to(x.dtype)
        # ---- backward ----
        dy_in = self._a2a(dy[flat_t[order]], ss, rs)[perm]
        dxs, dgs = [], []
        dw1 = torch.empty_like(self.w1)
        dw2 = torch.empty_like(self.w2)
        off = 0
        for j in range(el):
            c = counts[j]
            xe, a, b, z = saved[j]
            d_out = dy_in[off:off + c]
            dz = d_out @ self.w2[j]
            dw2[j] = d_out.T @ z
            g = gs[off:off + c, None].to(a.dtype)
            sb = torch.sigmoid(b.float())
            da = dz.float() * g.float() * b.float() * sb
            db = dz.float() * g.float() * a.float() * sb * (1 + b.float() * (1 - sb))
            dgs.append((dz.float() * a.float() * b.float() * sb).sum(1))
            dh1 = torch.cat([da, db], 1).to(x.dtype)
            dw1[j] = dh1.T @ xe
            dxs.append(dh1 @ self.w1[j])
            off += c
        dxr = torch.cat(dxs) if dxs else xs.new_zeros(0, self.h)
        dgr = torch.cat(dgs) if dgs else xs.new_zeros(0, dtype=torch.float32)
        b1 = torch.empty_like(dxr)
        b1[perm] = dxr
        b2 = torch.empty_like(dgr)
        b2[perm] = dgr
        dx_rows = self._a2a(b1, rs, ss)
        dg_rows = self._a2a(b2, rs, ss)
        dx = torch.zeros(Tr, self.h, dtype=torch.float32, device=x.device)
        dx.index_add_(0, flat_t[order], dx_rows.float())
        dgates = torch.zeros(Tr * k, dtype=torch.float32, device=x.device)
        dgates[order] = dg_rows
        dgates = dgates.view(Tr, k)
        dl_sel = gates * (dgates - (gates * dgates).sum(1, keepdim=True))
        dlogits = torch.zeros_like(logits).scatter_(1, topi, dl_sel)
        dx += dlogits @ self.wr.float()
        dwr = dlogits.T @ x.float()
        return y, dx.to(x.dtype), dw1, dw2, dwr


class NcclMoEGroupedBaseline(NcclMoEBaseline):
    """The stronger library baseline: the same NCCL all_to_all dispatch /
    combine, with every expert GEMM as ONE torch._grouped_mm call (CUTLASS
    grouped GEMM; measured within ±5% of this repo's plain grouped GEMM, see
    bench.py gemm_vs_cublas) and the SwiGLU / gate backward in bf16 torch ops.
    What separates it from the fused layer is then only the fusion (scatter,
    SwiGLU, gather and the NVLink exchange inside the GEMMs) and the overlap."""

    def step(self, x, dy):
        Tr, k, E, el, n, f = self.Tr, self.k, self.E, self.el, self.n, self.f
        logits = (x @ self.wr.T).float()
        topv, topi = logits.topk(k, dim=1)
        gates = torch.softmax(topv, dim=1)
        flat_e = topi.flatten()
        flat_t = torch.arange(Tr, device=x.device).repeat_interleave(k)
        order = torch.argsort(flat_e, stable=True)
        dest = flat_e[order] // el
        send = torch.bincount(dest, minlength=n)
        recv = torch.empty_like(send)
        if n > 1:
            dist.all_to_all_single(recv, send)
        else:
            recv = send
        ss, rs = send.tolist(), recv.tolist()
        xin = self._a2a(x[flat_t[order]], ss, rs)
        e_in = self._a2a(flat_e[order].to(torch.int32), ss, rs)
        g_in = self._a2a(gates.flatten()[order], ss, rs)
        perm = torch.argsort(e_in, stable=True)
        xs, es, gs = xin[perm], e_in[perm], g_in[perm]
        counts = torch.bincount(es.long() - self.rank * el, minlength=el)
        offs = counts.cumsum(0).to(torch.int32)
        g = gs[:, None].to(x.dtype)
        # forward: fc1 (gate+up), SwiGLU * gate, fc2 — one grouped GEMM each
        h1 = torch._grouped_mm(xs, self.w1.transpose(1, 2), offs=offs)
        a, b = h1[:, :f], h1[:, f:]
        sb = torch.sigmoid(b)
        z = a * (b * sb) * g
        out = torch._grouped_mm(z, self.w2.transpose(1, 2), offs=offs)
        back = torch.empty_like(out)
        back[perm] = out
        ret = self._a2a(back, rs, ss)
        y = torch.zeros(Tr, self.h, dtype=torch.float32, device=x.device)
        y.index_add_(0, flat_t[order], ret.float())
        y = y.to(x.dtype)
        # backward
        dy_in = self._a2a(dy[flat_t[order]], ss, rs)[perm]
        dz = torch._grouped_mm(dy_in, self.w2, offs=offs)
        dw2 = torch._grouped_mm(dy_in.t(), z, offs=offs)
        silu = b * sb
        dg = (dz * a * silu).float().sum(1)
        da = dz * g * silu
        db = dz * g * a * (sb * (1 + b * (1 - sb)))
        dh1 = torch.cat([da, db], 1)
        dw1 = torch._grouped_mm(dh1.t(), xs, offs=offs)
        dxr = torch._grouped_mm(dh1, self.w1, offs=offs)
        b1 = torch.empty_like(dxr)
        b1[perm] = dxr
        b2 = torch.empty_like(dg)
        b2[perm] = dg
        dx_rows = self._a2a(b1, rs, ss)
        dg_rows = self._a2a(b2, rs, ss)
        dx = torch.zeros(Tr, self.h, dtype=torch.float32, device=x.device)
        dx.index_add_(0, flat_t[order], dx_rows.float())
        dgates = torch.zeros(Tr * k, dtype=torch.float32, device=x.device)
        dgates[order] = dg_rows
        dgates = dgates.view(Tr, k)
        dl_sel = gates * (dgates - (gates * dgates).sum(1, keepdim=True))
        dlogits = torch.zeros_like(logits).scatter_(1, topi, dl_sel)
        dx += dlogits @ self.wr.float()
        dwr = dlogits.T @ x.float()
        return y, dx.to(x.dtype), dw1, dw2, dwr
