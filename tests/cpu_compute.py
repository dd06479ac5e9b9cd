"""CPU stand-in for the tile kernels, injected into the strategies by the
world-size>1 gloo tests ONLY (the product path calls the CUDA extension).

Same contracts as paper_2503_15758_b200.ops: [bh, rows, h] views, index maps
carrying global token positions, partial (O fp32, LSE) outputs, accumulate
mode, unscaled dq_acc accumulation.  Arithmetic in float64, restating the
reference's dense algebra (attention.py:127-160)."""

from __future__ import annotations

import torch


def _scores(q, k, causal, scale, q_index, k_index):
    s = torch.einsum("bqh,bkh->bqk", q.double(), k.double()) * scale
    if causal:
        qi = torch.as_tensor(q_index.host())
        ki = torch.as_tensor(k_index.host())
        s = s.masked_fill(~(qi[:, None] >= ki[None, :]), float("-inf"))
    return s


def _lse(s):
    lse = torch.logsumexp(s, dim=-1)
    safe = torch.where(torch.isinf(lse), torch.zeros_like(lse), lse)
    return lse, torch.exp(s - safe[..., None])


def tile_forward(q, k, v, *, causal, scale, q_index=None, k_index=None, out=None, lse=None,
                 out_dtype=torch.float32, accumulate=False):
    s = _scores(q, k, causal, scale, q_index, k_index)
    lse_new, p = _lse(s)
    o_new = torch.einsum("bqk,bkh->bqh", p, v.double())
    if accumulate:
        lse_old = lse.double()
        mx = torch.maximum(lse_old, lse_new)
        safe = torch.where(torch.isinf(mx), torch.zeros_like(mx), mx)
        wo = torch.where(torch.isneginf(lse_old), torch.zeros_like(mx), torch.exp(lse_old - safe))
        wn = torch.where(torch.isneginf(lse_new), torch.zeros_like(mx), torch.exp(lse_new - safe))
        tot = wo + wn
        o_new = (out.double() * wo[..., None] + o_new * wn[..., None]) / torch.where(
            tot > 0, tot, torch.ones_like(tot))[..., None]
        lse_new = torch.where(tot > 0, safe + torch.log(torch.where(tot > 0, tot, torch.ones_like(tot))),
                              torch.full_like(tot, float("-inf")))
    out.copy_(o_new.to(out.dtype))
    lse.copy_(lse_new.to(lse.dtype))
    return out, lse


def lse_merge(o_parts, lse_parts, *, out=None, lse_out=None, out_dtype=torch.bfloat16):
    lp = lse_parts.double()
    mx = lp.max(dim=0).values
    safe = torch.where(torch.isinf(mx), torch.zeros_like(mx), mx)
    w = torch.where(torch.isneginf(lp), torch.zeros_like(lp), torch.exp(lp - safe))
    tot = w.sum(0)
    o = torch.einsum("kr,krh->rh", w, o_parts.double()) / torch.where(
        tot > 0, tot, torch.ones_like(tot))[:, None]
    lse = torch.where(tot > 0, safe + torch.log(torch.where(tot > 0, tot, torch.ones_like(tot))),
                      torch.full_like(tot, float("-inf")))
    return o.to(out_dtype), lse.float()


def bwd_preprocess(o, dout):
    return (o.double() * dout.double()).sum(-1).float().contiguous()


def tile_backward(q, k, v, dout, lse, delta, *, causal, scale, q_index=None, k_index=None,
                  dq_acc=None, dk=None, dv=None, dkv_dtype=torch.float32, accumulate_dkv=False):
    s = _scores(q, k, causal, scale, q_index, k_index)
    l = lse.double()
    p = torch.exp(s - torch.where(torch.isinf(l), torch.full_like(l, float("inf")), l)[..., None])
    dp = torch.einsum("bqh,bkh->bqk", dout.double(), v.double())
    ds = p * (dp - delta.double()[..., None])
    dq_acc.add_(torch.einsum("bqk,bkh->bqh", ds, k.double()).to(dq_acc.dtype))
    gk = torch.einsum("bqk,bqh->bkh", ds, q.double()) * scale
    gv = torch.einsum("bqk,bqh->bkh", p, dout.double())
    if accumulate_dkv:
        gk, gv = gk + dk.double(), gv + dv.double()
    dk.copy_(gk.to(dk.dtype))
    dv.copy_(gv.to(dv.dtype))
    return dq_acc, dk, dv


def bwd_finalize(dq_acc, scale, out=None, dtype=torch.bfloat16):
    if out is None:
        out = torch.empty(dq_acc.shape, dtype=dtype)
    out.copy_((dq_acc.double() * scale).to(out.dtype))
    return out
