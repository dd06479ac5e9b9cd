"""Exact attention building blocks with the reference's names and contracts
(reference pkg/src/attn2d/attention.py), computed by the sm_100a kernels.

A partial result is kept in its unique (O, LSE) form on the device; the
reference's (m, n, d) triple is exposed as views (m = LSE, d = 1 for live
rows, n = O d), so `attn_fix` / `finalize` / `logsumexp` keep their meaning.
Inputs may be numpy arrays or torch tensors; they are rounded once to bf16
(the kernels' input precision) and results come back as fp32 CUDA tensors.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import ops
from .errors import FullyMaskedRowError, ShapeError, UnsupportedError


class MaskKind(str, Enum):
    NONE = "none"
    CAUSAL = "causal"
    ADDITIVE = "additive"


@dataclass(frozen=True)
class MaskSpec:
    """Masking rule (attention.py:27-47)."""

    kind: MaskKind = MaskKind.NONE
    additive: object | None = None

    def __post_init__(self):
        if self.kind is MaskKind.ADDITIVE and self.additive is None:
            raise ShapeError("additive mask requires a matrix")
        if self.kind is not MaskKind.ADDITIVE and self.additive is not None:
            raise ShapeError(f"mask kind {self.kind.value!r} takes no matrix")

    @classmethod
    def none(cls) -> "MaskSpec":
        return cls(MaskKind.NONE)

    @classmethod
    def causal(cls) -> "MaskSpec":
        return cls(MaskKind.CAUSAL)


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def _as_matrix(a, name="matrix") -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))
    if t.dim() != 2:
        raise ShapeError(f"expected a 2-D {name}, got shape {tuple(t.shape)}")
    return t


@dataclass
class TokenShard:
    """Rows of a global (n, h) tensor with their strictly increasing global
    positions (attention.py:50-72)."""

    data: object
    indices: object

    def __post_init__(self):
        self.data = _as_matrix(self.data, "shard")
        idx = self.indices
        if isinstance(idx, torch.Tensor):
            idx = idx.cpu().numpy()
        self.indices = np.asarray(idx, dtype=np.int64)
        if self.indices.ndim != 1 or len(self.indices) != self.data.shape[0]:
            raise ShapeError(f"{len(self.indices)} indices for {self.data.shape[0]} rows")
        if len(self.indices) > 1 and not np.all(np.diff(self.indices) > 0):
            raise ShapeError("shard indices must be strictly increasing")

    @property
    def rows(self) -> int:
        return self.data.shape[0]


@dataclass
class PartialAttn:
    """Streaming attention state for a fixed set of query rows
    (attention.py:75-110), held as (O normalised, LSE) on the device."""

    o: torch.Tensor    # (rows, h) fp32
    lse: torch.Tensor  # (rows,) fp32, -inf where nothing attended

    def __post_init__(self):
        if self.o.dim() != 2 or self.lse.shape != (self.o.shape[0],):
            raise ShapeError(f"inconsistent partial shapes o={tuple(self.o.shape)} "
                             f"lse={tuple(self.lse.shape)}")

    @classmethod
    def empty(cls, rows: int, h: int, device=None) -> "PartialAttn":
        dev = device or _device()
        return cls(torch.zeros((rows, h), dtype=torch.float32, device=dev),
                   torch.full((rows,), float("-inf"), dtype=torch.float32, device=dev))

    @property
    def rows(self) -> int:
        return self.o.shape[0]

    @property
    def m(self) -> torch.Tensor:
        return self.lse

    @property
    def d(self) -> torch.Tensor:
        return torch.isfinite(self.lse).to(torch.float32)

    @property
    def n(self) -> torch.Tensor:
        return self.o * self.d[:, None]

    @property
    def logsumexp(self) -> torch.Tensor:
        """m + log d, -inf for empty rows (attention.py:103-107)."""
        return self.lse

    def copy(self) -> "PartialAttn":
        return PartialAttn(self.o.clone(), self.lse.clone())


def _padded_h(h: int) -> int:
    """Head dim the kernels run: h rounded up to a multiple of 8 (16-byte
    rows; the tiles zero-fill the rest of their 64 / 128 columns)."""
    if h <= 128:
        return max(8, -(-h // 8) * 8)
    raise UnsupportedError(f"head dim {h} > 128 is not supported by the sm_100a tile")


def _to_bf16(t: torch.Tensor, hp: int) -> torch.Tensor:
    t = t.to(device=_device(), dtype=torch.bfloat16)
    if t.shape[-1] != hp:
        t = torch.nn.functional.pad(t, (0, hp - t.shape[-1]))
    return t.contiguous()[None]


def _check_streaming_mask(mask: MaskSpec):
    if mask.kind is MaskKind.ADDITIVE:
        raise ShapeError("additive masks exist on the dense reference path only")


def flash_attn_forward(q: TokenShard, k: TokenShard, v: TokenShard,
                       mask: MaskSpec | None = None, scale: float = 1.0,
                       block: int = 64) -> PartialAttn:
    """Streaming attention of q against exactly the keys/values in k, v
    (attention.py:168-191).  `block` is validated for parity; the kernel's
    key block is 128 (results are block-invariant, test_kernels.py:112-122)."""
    mask = mask or MaskSpec.none()
    _check_streaming_mask(mask)
    if k.rows != v.rows or not np.array_equal(k.indices, v.indices):
        raise ShapeError("k and v shards must cover the same rows")
    if q.data.shape[1] != k.data.shape[1]:
        raise ShapeError(f"head dims differ: q {tuple(q.data.shape)} k {tuple(k.data.shape)}")
    if block < 1:
        raise ShapeError("block must be positive")
    h = v.data.shape[1]
    hp = _padded_h(max(h, q.data.shape[1]))
    if q.rows == 0:
        return PartialAttn.empty(0, h)
    if k.rows == 0:
        return PartialAttn.empty(q.rows, h)
    qi = ops.TokenIndex.from_indices(q.indices, _device())
    ki = ops.TokenIndex.from_indices(k.indices, _device())
    o, lse = ops.tile_forward(_to_bf16(q.data, hp), _to_bf16(k.data, hp), _to_bf16(v.data, hp),
                              causal=mask.kind is MaskKind.CAUSAL, scale=float(scale),
                              q_index=qi, k_index=ki)
    return PartialAttn(o[0, :, :h].contiguous(), lse[0])


def attn_fix(a: PartialAttn, b: PartialAttn) -> PartialAttn:
    """Merge two partials over disjoint key sets (attention.py:194-214) with
    the k-way LSE-merge kernel (k = 2)."""
    if a.o.shape != b.o.shape:
        raise ShapeError(f"partials disagree: {tuple(a.o.shape)} vs {tuple(b.o.shape)}")
    rows, h = a.o.shape
    if rows == 0:
        return a.copy()
    hp = (h + 3) // 4 * 4
    parts = torch.zeros((2, rows, hp), dtype=torch.float32, device=a.o.device)
    parts[0, :, :h] = a.o
    parts[1, :, :h] = b.o
    lses = torch.stack([a.lse, b.lse]).contiguous()
    o, lse = ops.lse_merge(parts, lses, out_dtype=torch.float32)
    return PartialAttn(o[:, :h].contiguous(), lse)


def finalize(p: PartialAttn) -> torch.Tensor:
    """Normalised output; a row that attended nothing is an error
    (attention.py:217-222)."""
    empty = torch.isneginf(p.lse)
    if bool(empty.any()):
        raise FullyMaskedRowError(
            f"rows {torch.nonzero(empty).flatten().tolist()} attended no keys")
    return p.o


def flash_attn_backward(q: TokenShard, k: TokenShard, v: TokenShard, o, d_out, m, d,
                        mask: MaskSpec | None = None, scale: float = 1.0):
    """Gradients of the rows of q against the key subset in k, v given the
    GLOBAL output and statistics (attention.py:225-257)."""
    mask = mask or MaskSpec.none()
    _check_streaming_mask(mask)
    if k.rows != v.rows or not np.array_equal(k.indices, v.indices):
        raise ShapeError("k and v shards must cover the same rows")
    o = _as_matrix(o, "o")
    d_out = _as_matrix(d_out, "d_out")
    m = m if isinstance(m, torch.Tensor) else torch.as_tensor(np.asarray(m))
    d = d if isinstance(d, torch.Tensor) else torch.as_tensor(np.asarray(d))
    h = v.data.shape[1]
    if tuple(o.shape) != (q.rows, h) or d_out.shape != o.shape:
        raise ShapeError(f"o/d_out shape {tuple(o.shape)}/{tuple(d_out.shape)} does not match q rows")
    if m.shape != (q.rows,) or d.shape != (q.rows,):
        raise ShapeError("statistics m, d must have one entry per query row")
    if q.data.shape[1] != k.data.shape[1]:
        raise ShapeError(f"head dims differ: q {tuple(q.data.shape)} k {tuple(k.data.shape)}")
    if bool((d == 0).any()):
        raise FullyMaskedRowError(
            f"rows {torch.nonzero(d == 0).flatten().tolist()} have empty statistics")
    dev = _device()
    if q.rows == 0 or k.rows == 0:  # nothing attends: zero gradients (attention.py:250-252)
        z = lambda r, c: torch.zeros((r, c), dtype=torch.float32, device=dev)  # noqa: E731
        return z(q.rows, q.data.shape[1]), z(k.rows, k.data.shape[1]), z(v.rows, h)
    hp = _padded_h(max(h, q.data.shape[1]))
    lse = (m.to(dev, torch.float64) + torch.log(d.to(dev, torch.float64))).to(torch.float32)
    qb, kb, vb = _to_bf16(q.data, hp), _to_bf16(k.data, hp), _to_bf16(v.data, hp)
    ob, dob = _to_bf16(o, hp), _to_bf16(d_out, hp)
    qi = ops.TokenIndex.from_indices(q.indices, dev)
    ki = ops.TokenIndex.from_indices(k.indices, dev)
    delta = ops.bwd_preprocess(ob, dob)
    dq_acc, dk, dv = ops.tile_backward(qb, kb, vb, dob, lse[None].contiguous(), delta,
                                       causal=mask.kind is MaskKind.CAUSAL, scale=float(scale),
                                       q_index=qi, k_index=ki)
    dq = dq_acc * float(scale)
    hq = q.data.shape[1]
    return dq[0, :, :hq], dk[0, :, :hq], dv[0, :, :h]


def count_unmasked(q_idx, k_idx, causal: bool) -> int:
    """Exact number of evaluated (q, k) pairs (attention.py:260-265) — the
    FLOP-accounting basis."""
    q_idx = np.asarray(q_idx)
    k_idx = np.asarray(k_idx)
    if not causal:
        return int(len(q_idx)) * int(len(k_idx))
    return int(np.searchsorted(np.sort(k_idx), q_idx, side="right").sum())
