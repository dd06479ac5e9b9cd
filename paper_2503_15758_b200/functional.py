"""Single-device exact attention as a torch.autograd.Function — the 1x1 grid
of Attention2D: one tile forward (finalize fused, 16-bit O + fp32 LSE saved)
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
        o, lse = ops.tile_forward(q, k, v, causal=causal, scale=scale, out_dtype=q.dtype)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.causal, ctx.scale = causal, scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        do = do.to(q.dtype)
        if do.stride(-1) != 1:
            do = do.contiguous()
        dq, dk, dv = attention_backward(q, k, v, o, lse, do, ctx.causal, ctx.scale)
        return dq, dk, dv, None, None


def attention_backward(q, k, v, o, lse, do, causal: bool, scale: float,
                       dq_acc: torch.Tensor | None = None):
    """(dq, dk, dv) in q's dtype (bf16 or fp16) for [bh, n, h] operands (k/v may have bh / g
    heads: GQA / MQA, their gradients summed over each group of g query
    heads in fp32)."""
    delta = ops.bwd_preprocess(o, do)
    if dq_acc is None:
        dq_acc = torch.zeros(q.shape, dtype=torch.float32, device=q.device)
    else:
        dq_acc.zero_()
    group = q.shape[0] // k.shape[0]
    dq_acc, dk, dv = ops.tile_backward(q, k, v, do, lse, delta, causal=causal, scale=scale,
                                       dq_acc=dq_acc,
                                       dkv_dtype=q.dtype if group == 1 else torch.float32)
    if group > 1:
        dk, dv = (t.view(k.shape[0], group, *t.shape[1:]).sum(1).to(q.dtype) for t in (dk, dv))
    dq = ops.bwd_finalize(dq_acc, scale, dtype=q.dtype)
    return dq, dk, dv


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, causal: bool = False,
              scale: float | None = None) -> torch.Tensor:
    """softmax(scale q k^T [+ causal]) v for q of shape [B, M, N, H] or
    [BH, N, H], bf16 or fp16, on one B200 (output and gradients in the
    input dtype).  k/v have the same shape, or M_kv heads
    with M_kv dividing M (grouped-query / multi-query attention: query head
    m reads k/v head m // (M / M_kv)).  scale defaults to 1/sqrt(H)."""
    if q.dim() not in (3, 4) or k.shape != v.shape or k.dim() != q.dim():
        raise ShapeError(f"q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)} do not conform")
    hd = 1 if q.dim() == 4 else 0
    if (q.shape[:hd] != k.shape[:hd] or q.shape[hd + 1:] != k.shape[hd + 1:]
            or k.shape[hd] < 1 or q.shape[hd] % k.shape[hd]):
        raise ShapeError(f"q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)} do not conform")
    h = q.shape[-1]
    if scale is None:
        scale = h ** -0.5
    if h > 128:
        raise ShapeError(f"head dim {h} > 128 is not supported")
    hp = max(8, -(-h // 8) * 8)
    if h != hp:
        # the kernels take any multiple of 8 up to 128 (the reference's 80 / 96
        # presets run natively, costmodel.py:73-79); other widths are zero-
        # padded to the next multiple of 8 and the extra columns sliced off
        pad = lambda x: torch.nn.functional.pad(x, (0, hp - h))  # noqa: E731
        return attention(pad(q), pad(k), pad(v), causal, scale)[..., :h]
    shp = q.shape
    if q.dim() == 4:
        q, k, v = (x.reshape(-1, x.shape[2], h) for x in (q, k, v))
    o = _TileAttention.apply(q, k, v, bool(causal), float(scale))
    return o.reshape(shp)
