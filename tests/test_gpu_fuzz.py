"""Seeded random sweep of the tile kernels against a torch fp32 restatement:
ragged row counts on both sides, head dims 8..128, bf16 and fp16 operands,
GQA / MQA groups,
global-index maps (offset and strided affine maps, blocked cyclic maps,
explicit index arrays, an array query map against an affine key map), causal and not, fp32 / bf16 outputs, rows with no
visible key.  The backward is fed the reference's own (LSE, delta), so it
is checked in isolation (numpy_backend.py:46-62 semantics: P from global
statistics, rows with LSE = -inf contribute nothing).  Tolerances as
SURVEY.md §8c: rel-Fro <= 1e-2, LSE max-abs <= 1e-3."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from gpu_util import max_abs, rel_fro

pytestmark = pytest.mark.gpu

REL_TOL = 1e-2
LSE_TOL = 1e-3
N_CASES = 100


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_15758_b200 import ops as _ops
    return _ops


def _maps(rng, ops, kind):
    """(nq, nk, q TokenIndex, k TokenIndex, q global idx, k global idx)."""
    TI = ops.TokenIndex
    if kind == "offset":
        nq, nk = int(rng.integers(1, 600)), int(rng.integers(1, 600))
        qb, kb = int(rng.integers(0, 400)), int(rng.integers(0, 400))
        qi, ki = TI.contiguous(nq, qb), TI.contiguous(nk, kb)
    elif kind == "strided":
        s = int(rng.integers(2, 4))
        nq, nk = int(rng.integers(1, 500)), int(rng.integers(1, 500))
        qi = TI(n=nq, bases=(int(rng.integers(0, s)),), stride=s, rows_per_block=nq)
        ki = TI(n=nk, bases=(int(rng.integers(0, s)),), stride=s, rows_per_block=nk)
    elif kind == "blocked":
        p = int(rng.choice([2, 4]))
        nbq, nbk = int(rng.integers(1, 3)), int(rng.integers(1, 3))
        rq, rk = 128 * int(rng.integers(1, 3)), 128 * int(rng.integers(1, 3))
        qi = TI.blocked([int(rng.integers(0, p)) + b * p * rq for b in range(nbq)], p, rq)
        ki = TI.blocked([int(rng.integers(0, p)) + b * p * rk for b in range(nbk)], p, rk)
        nq, nk = qi.n, ki.n
    elif kind == "mixed":  # explicit query subset against an offset key range
        nq, nk = int(rng.integers(1, 400)), int(rng.integers(1, 600))
        qg = np.sort(rng.choice(1500, nq, replace=False)).astype(np.int64)
        qi, ki = TI.from_indices(qg), TI.contiguous(nk, int(rng.integers(0, 800)))
    else:  # array
        nq, nk = int(rng.integers(1, 500)), int(rng.integers(1, 500))
        qg = np.sort(rng.choice(2000, nq, replace=False)).astype(np.int64)
        kg = np.sort(rng.choice(2000, nk, replace=False)).astype(np.int64)
        qi, ki = TI.from_indices(qg), TI.from_indices(kg)
    return nq, nk, qi, ki, torch.from_numpy(qi.host().copy()), torch.from_numpy(ki.host().copy())


def _reference(q, k, v, dout, causal, scale, qg, kg, group):
    """fp32 forward (O, LSE) and backward (dQ, dK, dV per query head)."""
    kf = k.float().repeat_interleave(group, 0)
    vf = v.float().repeat_interleave(group, 0)
    qf, df = q.float(), dout.float()
    s = torch.einsum("bqh,bkh->bqk", qf, kf) * scale
    if causal:
        mask = qg.cuda()[:, None] >= kg.cuda()[None, :]
        s = s.masked_fill(~mask, float("-inf"))
    lse = torch.logsumexp(s, dim=-1)
    safe = torch.where(torch.isinf(lse), torch.zeros_like(lse), lse)
    p = torch.exp(s - safe[..., None])
    o = torch.einsum("bqk,bkh->bqh", p, vf)
    delta = (df * o).sum(-1)
    dp = torch.einsum("bqh,bkh->bqk", df, vf)
    ds = p * (dp - delta[..., None])
    dq = torch.einsum("bqk,bkh->bqh", ds, kf) * scale
    dk = torch.einsum("bqk,bqh->bkh", ds, qf) * scale
    dv = torch.einsum("bqk,bqh->bkh", p, df)
    return o, lse, delta, dq, dk, dv


def _close(got, want, what, tag):
    # relative where the result has magnitude; absolute where it is pure
    # rounding noise (e.g. dQ = 0 exactly with a single visible key)
    err = max_abs(got, want)
    assert err < 1e-5 or rel_fro(got, want) < REL_TOL, (tag, what, rel_fro(got, want), err)


@pytest.mark.parametrize("case", range(N_CASES))
def test_random_tile_calls_match_torch(ops, case):
    rng = np.random.default_rng(1000 + case)
    kind = ["offset", "strided", "blocked", "array", "mixed"][case % 5]
    nq, nk, qi, ki, qg, kg = _maps(rng, ops, kind)
    h = int(rng.choice([8, 16, 40, 64, 72, 96, 120, 128]))
    group = int(rng.choice([1, 1, 2, 4]))
    bh_kv = int(rng.integers(1, 3))
    bh = bh_kv * group
    causal = bool(rng.integers(0, 2))
    scale = float(rng.choice([h ** -0.5, 1.0]))
    dt = torch.float16 if rng.integers(0, 3) == 0 else torch.bfloat16  # operand type
    out_dtype = torch.float32 if rng.integers(0, 2) else dt
    tag = dict(kind=kind, nq=nq, nk=nk, h=h, group=group, bh=bh, causal=causal, scale=scale,
               dt=str(dt), out=str(out_dtype))
    g = torch.Generator(device="cpu").manual_seed(case)

    def rnd(*shape):
        return (torch.rand(shape, generator=g) * 2 - 1).to(device="cuda", dtype=dt)

    q, dout = rnd(bh, nq, h), rnd(bh, nq, h)
    k, v = rnd(bh_kv, nk, h), rnd(bh_kv, nk, h)
    o_ref, lse_ref, delta, dq_ref, dk_ref, dv_ref = _reference(q, k, v, dout, causal, scale,
                                                               qg, kg, group)
    o, lse = ops.tile_forward(q, k, v, causal=causal, scale=scale, q_index=qi, k_index=ki,
                              out_dtype=out_dtype)
    torch.cuda.synchronize()
    seen = torch.isfinite(lse_ref)
    assert torch.equal(torch.isfinite(lse), seen), tag
    if bool(seen.any()):
        assert max_abs(lse[seen], lse_ref[seen]) < LSE_TOL, (tag, max_abs(lse[seen], lse_ref[seen]))
    if bool((~seen).any()):  # rows that attended nothing: O = 0
        assert float(o.float()[~seen].abs().max()) == 0.0, tag
    _close(o.float(), o_ref, "O", tag)

    dq_acc, dk, dv = ops.tile_backward(q, k, v, dout, lse_ref.contiguous(), delta.contiguous(),
                                       causal=causal, scale=scale, q_index=qi, k_index=ki)
    torch.cuda.synchronize()
    _close(dq_acc * scale, dq_ref, "dQ", tag)
    _close(dk, dk_ref, "dK", tag)
    _close(dv, dv_ref, "dV", tag)
