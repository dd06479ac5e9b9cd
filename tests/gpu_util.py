"""Shared helpers for the GPU parity tests (torch fp32 reference of the same
op, seeded inputs per the reference convention cli.py:56-61)."""

from __future__ import annotations

import numpy as np
import torch


def bf16_from_bits(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(bits.astype(np.int16).view(np.int16)).view(torch.bfloat16)


def uniform(shape, seed, device="cuda"):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.rand(shape, generator=g) * 2 - 1).to(device=device, dtype=torch.bfloat16)


def ref_attention(q, k, v, causal, scale, q_idx=None, k_idx=None):
    """fp32 reference: softmax(scale q k^T, causal by global index) v and LSE.
    q [bh, nq, h], k/v [bh, nk, h]; returns (o fp32, lse fp32)."""
    qf, kf, vf = q.float(), k.float(), v.float()
    s = torch.einsum("bqh,bkh->bqk", qf, kf) * scale
    if causal:
        nq, nk = q.shape[1], k.shape[1]
        qi = torch.arange(nq, device=q.device) if q_idx is None else q_idx.to(q.device)
        ki = torch.arange(nk, device=q.device) if k_idx is None else k_idx.to(q.device)
        mask = qi[:, None] >= ki[None, :]
        s = s.masked_fill(~mask, float("-inf"))
    lse = torch.logsumexp(s, dim=-1)
    p = torch.exp(s - torch.where(torch.isinf(lse), torch.zeros_like(lse), lse)[..., None])
    o = torch.einsum("bqk,bkh->bqh", p, vf)
    return o, lse


def ref_attention_grad(q, k, v, dout, causal, scale):
    qf = q.float().requires_grad_(True)
    kf = k.float().requires_grad_(True)
    vf = v.float().requires_grad_(True)
    o, _ = ref_attention(qf, kf, vf, causal, scale)
    o.backward(dout.float())
    return qf.grad, kf.grad, vf.grad


def rel_fro(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def max_abs(a, b):
    return float((a.double() - b.double()).abs().max())
