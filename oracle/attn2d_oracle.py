"""CPU oracle for the Attention2D hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference's algorithm for the
path `north_star` names (tile forward/backward, the partial-softmax merge,
finalize, the dense oracle and the cyclic layouts).  It exists so that
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs have a checker and a CPU timing arm.  The product
path (`paper_2503_15758_b200`) never imports it; the CUDA extension is the
only implementation shipped.

Parity pinning: the restatement is checked against golden vectors produced
by importing the reference package itself (`tests/golden/make_golden.py`,
fixtures in `tests/golden/*.npz`) and against the reference's own
known-answer tests, see `tests/test_oracle.py`.

Every function cites the reference file:line it follows (paths relative to
the reference's `pkg/src/attn2d/`).
"""

from __future__ import annotations

import numpy as np

# Key/value chunk of the backward recurrence (kernels/numpy_backend.py:11-13).
_BWD_CHUNK = 128


# ---------------------------------------------------------------------------
# Tile kernels (kernels/numpy_backend.py:24-62, kernels/__init__.py:70-92)
# ---------------------------------------------------------------------------

def flash_forward(q, k, v, q_idx, k_idx, causal, scale, block, m, nacc, d):
    """Streaming (m, n, d) recurrence over key blocks, updated in place.

    Follows kernels/numpy_backend.py:24-43: per key block, scores are
    masked by *global* index (q_idx >= k_idx), m_new = max(m, rowmax),
    alpha = exp(m - m_new), rows that have attended nothing stay empty.
    """
    nk = k.shape[0]
    st = q.dtype.type(scale)
    for start in range(0, nk, block):
        stop = min(start + block, nk)
        s = (q @ k[start:stop].T) * st
        if causal:
            s = np.where(q_idx[:, None] >= k_idx[None, start:stop], s, -np.inf)
        m_new = np.maximum(m, s.max(axis=1))
        live = m_new > -np.inf
        with np.errstate(invalid="ignore"):
            alpha = np.exp(m - m_new)
            w = np.exp(s - m_new[:, None])
        alpha[~live] = 0.0
        w[~live, :] = 0.0
        d[:] = alpha * d + w.sum(axis=1)
        nacc[:] = alpha[:, None] * nacc + w @ v[start:stop]
        m[:] = np.where(live, m_new, m)


def flash_backward(q, k, v, o, d_out, m_stat, d_stat, q_idx, k_idx, causal,
                   scale, dq, dk, dv):
    """Accumulate (dq, dk, dv) for a key subset from global row statistics.

    Follows kernels/numpy_backend.py:46-62: delta = rowsum(dO*O),
    P = exp(s - m)/d, dV += P^T dO, dS = P*(dO V^T - delta),
    dQ += dS K * scale, dK += dS^T Q * scale.
    """
    nk = k.shape[0]
    st = q.dtype.type(scale)
    delta = np.sum(d_out * o, axis=1)
    for start in range(0, nk, _BWD_CHUNK):
        stop = min(start + _BWD_CHUNK, nk)
        kb, vb = k[start:stop], v[start:stop]
        s = (q @ kb.T) * st
        if causal:
            s = np.where(q_idx[:, None] >= k_idx[None, start:stop], s, -np.inf)
        p = np.exp(s - m_stat[:, None]) / d_stat[:, None]
        dv[start:stop] += p.T @ d_out
        dp = d_out @ vb.T
        ds = p * (dp - delta[:, None])
        dq += (ds @ kb) * st
        dk[start:stop] += (ds.T @ q) * st


# ---------------------------------------------------------------------------
# Partial-softmax algebra (attention.py:75-110, :194-222)
# ---------------------------------------------------------------------------

def empty_partial(rows, h, dtype=np.float64):
    """PartialAttn.empty (attention.py:91-97): (m=-inf, n=0, d=0)."""
    return (np.full(rows, -np.inf, dtype=dtype), np.zeros((rows, h), dtype=dtype),
            np.zeros(rows, dtype=dtype))


def logsumexp(m, d):
    """PartialAttn.logsumexp (attention.py:103-107): m + log d, -inf if d == 0."""
    with np.errstate(divide="ignore"):
        return np.where(d > 0, m + np.log(d), -np.inf)


def attn_fix(a, b):
    """Associative merge of two partials (attention.py:194-214)."""
    am, an, ad = a
    bm, bn, bd = b
    m = np.maximum(am, bm)
    both_empty = np.isneginf(m)
    with np.errstate(invalid="ignore"):
        ea = np.exp(am - m)
        eb = np.exp(bm - m)
    ea[both_empty] = 0.0
    eb[both_empty] = 0.0
    return m, ea[:, None] * an + eb[:, None] * bn, ea * ad + eb * bd


def finalize(part):
    """n / d; a zero denominator is an error (attention.py:217-222,
    linalg.py:59-71)."""
    _, n, d = part
    if np.any(d == 0):
        raise ZeroDivisionError("rows attended no keys")
    return n / d[:, None]


def lse_merge(o_parts, lse_parts):
    """k-way merge in (normalised O, LSE) form — the same algebra as a fold
    of attn_fix with (m, n, d) = (lse, o, 1)."""
    lse = np.stack(lse_parts)                      # (k, rows)
    mx = np.max(lse, axis=0)
    safe = np.where(np.isneginf(mx), 0.0, mx)
    w = np.exp(lse - safe[None, :])                # empty partials weigh 0
    tot = w.sum(axis=0)
    with np.errstate(invalid="ignore", divide="ignore"):
        o = np.einsum("kr,krh->rh", w, np.stack(o_parts)) / tot[:, None]
        out_lse = np.where(tot > 0, safe + np.log(tot), -np.inf)
    o[tot == 0] = 0.0
    return o, out_lse


# ---------------------------------------------------------------------------
# Dense oracle (attention.py:113-160) and work accounting (:260-265)
# ---------------------------------------------------------------------------

def _dense_scores(q, k, causal, scale, q_idx=None, k_idx=None):
    s = (q @ k.T) * q.dtype.type(scale)
    qi = np.arange(q.shape[0]) if q_idx is None else np.asarray(q_idx)
    ki = np.arange(k.shape[0]) if k_idx is None else np.asarray(k_idx)
    if causal:
        s = np.where(qi[:, None] >= ki[None, :], s, -np.inf)
    return s


def reference_attention(q, k, v, causal=False, scale=1.0, q_idx=None, k_idx=None):
    """softmax(scale q k^T + mask) v, max-subtracted (attention.py:127-142)."""
    s = _dense_scores(q, k, causal, scale, q_idx, k_idx)
    m = s.max(axis=1)
    if np.any(np.isneginf(m)):
        raise ZeroDivisionError("fully masked row")
    e = np.exp(s - m[:, None])
    return (e / e.sum(axis=1)[:, None]) @ v


def reference_lse(q, k, causal=False, scale=1.0, q_idx=None, k_idx=None):
    s = _dense_scores(q, k, causal, scale, q_idx, k_idx)
    m = s.max(axis=1)
    with np.errstate(invalid="ignore", divide="ignore"):
        return m + np.log(np.exp(s - m[:, None]).sum(axis=1))


def reference_attention_grad(q, k, v, d_out, causal=False, scale=1.0):
    """Dense analytic gradients (attention.py:145-160)."""
    s = _dense_scores(q, k, causal, scale)
    m = s.max(axis=1)
    e = np.exp(s - m[:, None])
    p = e / e.sum(axis=1)[:, None]
    o = p @ v
    dv = p.T @ d_out
    dp = d_out @ v.T
    ds = p * (dp - np.sum(d_out * o, axis=1)[:, None])
    st = q.dtype.type(scale)
    return (ds @ k) * st, (ds.T @ q) * st, dv


def count_unmasked(q_idx, k_idx, causal):
    """Exact evaluated (q, k) pairs (attention.py:260-265)."""
    if not causal:
        return int(len(q_idx)) * int(len(k_idx))
    ks = np.sort(np.asarray(k_idx))
    return int(np.searchsorted(ks, np.asarray(q_idx), side="right").sum())


# ---------------------------------------------------------------------------
# Layouts (layouts.py:53-65, strategies/ring.py:27-38)
# ---------------------------------------------------------------------------

def cyclic_indices(n, p, form, r, c):
    """CyclicLayout.indices for a square grid (layouts.py:53-65)."""
    side = int(round(p ** 0.5))
    if form == "column_major":
        return np.arange(r + side * c, n, p, dtype=np.int64)
    if form == "row_major":
        return np.arange(side * r + c, n, p, dtype=np.int64)
    if form == "row_gathered":
        return np.arange(r, n, side, dtype=np.int64)
    return np.arange(c, n, side, dtype=np.int64)


def ring_block_indices(n, p, rank):
    """TE load-balanced ring rows (strategies/ring.py:27-38)."""
    if p == 1:
        return np.arange(n, dtype=np.int64)
    c = n // (2 * p)
    front = np.arange(rank * c, (rank + 1) * c, dtype=np.int64)
    back = np.arange(n // 2 + (p - 1 - rank) * c, n // 2 + (p - rank) * c, dtype=np.int64)
    return np.concatenate([front, back])


# ---------------------------------------------------------------------------
# Convenience: one full tile fwd/bwd over a whole head (used by the CPU arm)
# ---------------------------------------------------------------------------

def tile_forward_full(q, k, v, q_idx, k_idx, causal, scale, block=64):
    """flash_attn_forward + finalize + logsumexp for one head
    (attention.py:168-191 then :217-222 / :103-107)."""
    m, n, d = empty_partial(q.shape[0], v.shape[1], q.dtype)
    flash_forward(q, k, v, q_idx, k_idx, causal, scale, block, m, n, d)
    with np.errstate(invalid="ignore", divide="ignore"):
        o = np.where(d[:, None] > 0, n / np.where(d > 0, d, 1.0)[:, None], 0.0)
    return o, logsumexp(m, d), (m, d)


def tile_backward_full(q, k, v, o, d_out, m, d, q_idx, k_idx, causal, scale):
    """flash_attn_backward (attention.py:225-257)."""
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    flash_backward(q, k, v, o, d_out, m, d, q_idx, k_idx, causal, scale, dq, dk, dv)
    return dq, dk, dv


def attention_flops(n_q_k_pairs, h, heads=1, backward=True):
    """FLOP accounting of BASELINE.md §3: 4·H·U fwd, ×3.5 fwd+bwd."""
    f = 4.0 * h * n_q_k_pairs * heads
    return f * 3.5 if backward else f


# ---------------------------------------------------------------------------
# Exact schedule identities of the reference (costmodel.py:106-153)
# ---------------------------------------------------------------------------

def predicted_phase_words(strategy, n, h, p, phase_fwd, on_diagonal):
    """Words one processor sends in one phase (costmodel.py:106-136): square
    p = s^2 for the 2D schedules, (m, n, d) partials of h + 2 words, backward
    bundles (q, o, d_out, m, d) of 3h + 2 words."""
    rows = n // p
    if strategy == "ring":
        if phase_fwd:
            return 2 * rows * h * (p - 1)
        return 4 * rows * h * (p - 1) + (2 * rows * h if p > 1 else 0)
    side = int(round(p ** 0.5))
    assert side * side == p
    transpose = 0 if on_diagonal else 2 * rows * h
    if phase_fwd:
        return (transpose + (side - 1) * rows * h + 2 * (side - 1) * rows * h
                + (side - 1) * rows * (h + 2))
    return (transpose + (side - 1) * rows * (3 * h + 2) + 2 * (side - 1) * rows * h
            + (side - 1) * rows * h + 2 * (side - 1) * rows * h)


def predicted_phase_msgs(strategy, n, h, p, phase_fwd, on_diagonal):
    """Messages one processor sends in one phase (costmodel.py:139-153)."""
    if strategy == "ring":
        return (p - 1) if phase_fwd else (p - 1) + (1 if p > 1 else 0)
    side = int(round(p ** 0.5))
    return (0 if on_diagonal else 1) + (3 if phase_fwd else 4) * (side - 1)
