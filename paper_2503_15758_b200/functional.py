"""Single-device exact attention as a torch.autograd.Function — the 1x1 grid
of Attention2D: one tile forward (finalize fused, bf16 O + fp32 LSE saved)
and one tile backward.  The saved state is (Q, K, V, O, LSE), the LSE form of
the reference's SavedState (strategies/common.py:64-80; PAPER Alg. 1
SaveForBackprop)."""

from __future__ import annotations

import torch

from . import ops
from .errors import ShapeError


class _TileAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, causal: bool, scale: float):
        o, lse = ops.tile_forward(q, k, v, causal=causal, scale=scale, out_dtype=torch.bfloat16)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.causal, ctx.scale = causal, scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        do = do.to(torch.bfloat16)
        if do.stride(-1) != 1:
            do = do.contiguous()
        dq, dk, dv = attention_backward(q, k, v, o, lse, do, ctx.causal, ctx.scale)
        return dq, dk, dv, None, None


def attention_backward(q, k, v, o, lse, do, causal: bool, scale: float,
                       dq_acc: torch.Tensor | None = None):
    """(dq, dk, dv) in bf16 for [bh, n, h] operands."""
    delta = ops.bwd_preprocess(o, do)
    if dq_acc is None:
        dq_acc = torch.zeros(q.shape, dtype=torch.float32, device=q.device)
    else:
        dq_acc.zero_()
    dq_acc, dk, dv = ops.tile_backward(q, k, v, do, lse, delta, causal=causal, scale=scale,
                                       dq_acc=dq_acc, dkv_dtype=torch.bfloat16)
    dq = ops.bwd_finalize(dq_acc, scale, dtype=torch.bfloat16)
    return dq, dk, dv


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, causal: bool = False,
              scale: float | None = None) -> torch.Tensor:
    """softmax(scale q k^T [+ causal]) v for q/k/v of shape [B, M, N, H] or
    [BH, N, H], bf16, on one B200.  scale defaults to 1/sqrt(H)."""
    if q.dim() not in (3, 4) or q.shape != k.shape or k.shape != v.shape:
        raise ShapeError(f"q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)} do not conform")
    h = q.shape[-1]
    if scale is None:
        scale = h ** -0.5
    shp = q.shape
    if q.dim() == 4:
        q, k, v = (x.reshape(-1, x.shape[2], h) for x in (q, k, v))
    o = _TileAttention.apply(q, k, v, bool(causal), float(scale))
    return o.reshape(shp)
