"""Torch-level wrappers over the C ABI: device memory and streams come from
PyTorch, compute is the sm_100a kernels in libattn2d_b200.so.

Tensors are [bh, rows, h] (bh = flattened batch x heads) with unit stride
along h.  Index maps describe the GLOBAL token position of every local row
(the reference's TokenShard.indices, attention.py:50-72).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .errors import ShapeError, UnsupportedError


# --------------------------------------------------------------------------
# index maps
# --------------------------------------------------------------------------

@dataclass
class TokenIndex:
    """Global token indices of the rows of a local buffer.

    `bases` / `stride` / `rows_per_block` describe the affine-blocked form
    base[b] + stride * i; `array` (int64 CUDA tensor) the explicit form.
    """

    n: int
    bases: tuple = (0,)
    stride: int = 1
    rows_per_block: int = 0
    array: torch.Tensor | None = None
    _host: np.ndarray | None = field(default=None, repr=False)

    @classmethod
    def contiguous(cls, n: int, start: int = 0) -> "TokenIndex":
        return cls(n=n, bases=(int(start),), stride=1, rows_per_block=n)

    @classmethod
    def blocked(cls, bases: Sequence[int], stride: int, rows_per_block: int) -> "TokenIndex":
        bases = tuple(int(b) for b in bases)
        return cls(n=len(bases) * rows_per_block, bases=bases, stride=int(stride),
                   rows_per_block=int(rows_per_block))

    @classmethod
    def from_indices(cls, idx, device=None) -> "TokenIndex":
        """Affine-blocked form when the indices have one, else the array form."""
        host = np.asarray(idx.cpu() if isinstance(idx, torch.Tensor) else idx, dtype=np.int64)
        n = int(host.shape[0])
        if n == 0:
            return cls(n=0)
        if n == 1:
            return cls(n=1, bases=(int(host[0]),), stride=1, rows_per_block=1, _host=host)
        d = np.diff(host)
        if np.all(d == d[0]) and d[0] >= 1:
            return cls(n=n, bases=(int(host[0]),), stride=int(d[0]), rows_per_block=n, _host=host)
        # fewest blocks of 128*k rows sharing a stride
        for nb in range(2, _lib.MAX_BLOCKS + 1):
            if n % nb or (n // nb) % 128:
                continue
            rpb = n // nb
            blk = host.reshape(n // rpb, rpb)
            dd = np.diff(blk, axis=1)
            if np.all(dd == dd[0, 0]) and dd[0, 0] >= 1:
                return cls.blocked(blk[:, 0].tolist(), int(dd[0, 0]), rpb)
        dev = device if device is not None else "cuda"
        return cls(n=n, array=torch.as_tensor(host, device=dev), _host=host)

    @property
    def is_array(self) -> bool:
        return self.array is not None

    def host(self) -> np.ndarray:
        if self._host is None:
            if self.is_array:
                self._host = self.array.cpu().numpy()
            else:
                rpb = self.rows_per_block or self.n
                parts = [b + self.stride * np.arange(min(rpb, self.n - i * rpb), dtype=np.int64)
                         for i, b in enumerate(self.bases)]
                self._host = np.concatenate(parts) if parts else np.zeros(0, np.int64)
        return self._host

    def as_array(self, device) -> "TokenIndex":
        if self.is_array:
            return self
        return TokenIndex(n=self.n, array=torch.as_tensor(self.host(), device=device),
                          _host=self.host())

    def to_c(self) -> _lib.IndexMap:
        m = _lib.IndexMap()
        if self.is_array:
            m.mode = _lib.IDX_ARRAY
            m.nblocks = 1
            m.rows_per_block = self.n
            m.stride = 1
            m.idx = self.array.data_ptr()
            return m
        m.mode = _lib.IDX_AFFINE
        m.nblocks = len(self.bases)
        m.rows_per_block = self.rows_per_block if len(self.bases) > 1 else self.n
        m.stride = self.stride
        for i, b in enumerate(self.bases):
            m.base[i] = b
        return m


def _pair_maps(qi: TokenIndex, ki: TokenIndex, causal: bool, device):
    """Both sides must share the mode (and the stride when causal)."""
    if qi.is_array != ki.is_array or (causal and not qi.is_array and qi.stride != ki.stride):
        qi, ki = qi.as_array(device), ki.as_array(device)
    if not qi.is_array and len(qi.bases) > 1 and qi.rows_per_block % 128:
        qi, ki = qi.as_array(device), ki.as_array(device)
    if not ki.is_array and len(ki.bases) > 1 and ki.rows_per_block % 128:
        qi, ki = qi.as_array(device), ki.as_array(device)
    return qi, ki


# --------------------------------------------------------------------------
# helpers
# --------------------------------------------------------------------------

# kernels this module has launched (bench.py reports the count in the timed region)
LAUNCHES = [0]


def launches() -> int:
    return LAUNCHES[0]


def _kv_group(bh: int, k: torch.Tensor) -> int:
    """Query heads per key/value head (GQA / MQA)."""
    bk = k.shape[0] if k.dim() == 3 else 0
    if bh == 0 and bk == 0:
        return 1
    if bk < 1 or bh % bk:
        raise ShapeError(f"{bk} key/value heads do not divide {bh} query heads")
    return bh // bk


def _stream(t: torch.Tensor) -> int:
    LAUNCHES[0] += 1
    return torch.cuda.current_stream(t.device).cuda_stream


# 16-bit operand types of the tile kernels (tcgen05 kind::f16)
INPUT_DTYPES = (torch.bfloat16, torch.float16)


def _check3(name: str, t: torch.Tensor, dtype=None):
    """[bh, rows, h] CUDA tensor with unit stride along h, of `dtype` (or,
    when None, of one of the 16-bit input types)."""
    if not t.is_cuda:
        raise ShapeError(f"{name} must be a CUDA tensor")
    if t.dim() != 3:
        raise ShapeError(f"{name} must be [bh, rows, h], got {tuple(t.shape)}")
    if dtype is None and t.dtype not in INPUT_DTYPES:
        raise ShapeError(f"{name} must be torch.bfloat16 or torch.float16, got {t.dtype}")
    if dtype is not None and t.dtype != dtype:
        raise ShapeError(f"{name} must be {dtype} like the other operands, got {t.dtype}")
    if t.shape[2] > 0 and t.stride(2) != 1:
        raise ShapeError(f"{name} must have unit stride along h")


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return _lib.F32
    if dt == torch.bfloat16:
        return _lib.BF16
    if dt == torch.float16:
        return _lib.F16
    raise UnsupportedError(f"output dtype {dt} not supported")


# --------------------------------------------------------------------------
# kernels
# --------------------------------------------------------------------------

def tile_forward(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, causal: bool,
                 scale: float, q_index: TokenIndex | None = None,
                 k_index: TokenIndex | None = None, out: torch.Tensor | None = None,
                 lse: torch.Tensor | None = None, out_dtype: torch.dtype = torch.float32,
                 accumulate: bool = False):
    """Partial attention of q against exactly the keys in k/v.  k/v may hold
    fewer heads than q (GQA / MQA): query head b reads k/v head b // group.

    q/k/v are bf16 or fp16 (all alike).
    Returns (o, lse): o [bh, nq, h] (fp32 normalised partial, or final O in
    bf16 / fp16),
    lse [bh, nq] fp32, -inf where a row attended nothing.  With accumulate,
    (out, lse) hold a previous partial and are merged in place.
    """
    lib = _lib.load()
    _check3("q", q)
    _check3("k", k, q.dtype)
    _check3("v", v, q.dtype)
    bh, nq, h = q.shape
    nk = k.shape[1]
    group = _kv_group(bh, k)
    if k.shape != (bh // group, nk, h) or v.shape != k.shape:
        raise ShapeError(f"q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)} do not conform")
    qi = q_index if q_index is not None else TokenIndex.contiguous(nq)
    ki = k_index if k_index is not None else TokenIndex.contiguous(nk)
    if qi.n != nq or ki.n != nk:
        raise ShapeError("index maps do not match the row counts")
    qi, ki = _pair_maps(qi, ki, causal, q.device)
    if out is None:
        if accumulate:
            raise ShapeError("accumulate needs an existing (out, lse) state")
        out = torch.empty((bh, nq, h), dtype=out_dtype, device=q.device)
    if lse is None:
        lse = torch.empty((bh, nq), dtype=torch.float32, device=q.device)
    if out.shape != (bh, nq, h) or out.stride(2) != 1:
        raise ShapeError("out must be [bh, nq, h] with unit stride along h")
    if lse.shape != (bh, nq) or not lse.is_contiguous() or lse.dtype != torch.float32:
        raise ShapeError("lse must be a contiguous fp32 [bh, nq] tensor")
    if nk == 0 and not accumulate:
        out.zero_()
        lse.fill_(float("-inf"))
        return out, lse
    a = _lib.TileFwdArgs()
    a.q, a.k, a.v, a.o, a.lse = (q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                 lse.data_ptr())
    a.q_stride_bh, a.q_stride_row = q.stride(0), q.stride(1)
    a.k_stride_bh, a.k_stride_row = k.stride(0), k.stride(1)
    a.v_stride_bh, a.v_stride_row = v.stride(0), v.stride(1)
    a.o_stride_bh, a.o_stride_row = out.stride(0), out.stride(1)
    a.bh, a.nq, a.nk, a.h = bh, nq, nk, h
    a.causal = int(bool(causal))
    a.scale = float(scale)
    a.o_dtype = _dtype_code(out.dtype)
    a.accumulate = int(bool(accumulate))
    a.q_map, a.k_map = qi.to_c(), ki.to_c()
    a.kv_group = group
    a.in_dtype = _dtype_code(q.dtype)
    _lib.check(lib.a2d_tile_fwd(a, _stream(q)), "a2d_tile_fwd")
    return out, lse


def bwd_preprocess(o: torch.Tensor, dout: torch.Tensor) -> torch.Tensor:
    """delta = rowsum(dO * O) in fp32 (numpy_backend.py:49)."""
    lib = _lib.load()
    _check3("o", o)
    _check3("dout", dout, o.dtype)
    if o.shape != dout.shape:
        raise ShapeError("o and dout differ in shape")
    bh, n, h = o.shape
    delta = torch.empty((bh, n), dtype=torch.float32, device=o.device)
    _lib.check(lib.a2d_bwd_preprocess(o.data_ptr(), dout.data_ptr(), delta.data_ptr(),
                                      o.stride(0), o.stride(1), dout.stride(0), dout.stride(1),
                                      bh, n, h, _dtype_code(o.dtype), _stream(o)),
               "a2d_bwd_preprocess")
    return delta


def tile_backward(q, k, v, dout, lse, delta, *, causal: bool, scale: float,
                  q_index: TokenIndex | None = None, k_index: TokenIndex | None = None,
                  dq_acc: torch.Tensor | None = None, dk: torch.Tensor | None = None,
                  dv: torch.Tensor | None = None, dkv_dtype: torch.dtype = torch.float32,
                  accumulate_dkv: bool = False):
    """Gradient contributions of the keys in k/v for the rows of q, given the
    GLOBAL (lse, delta) statistics of those rows (attention.py:225-257).

    dq_acc (fp32, unscaled dS K) is accumulated into; dk (scaled) and dv are
    written, one per QUERY head (with GQA the caller sums each group), or,
    with accumulate_dkv, added to the fp32 dk / dv already there.
    Returns (dq_acc, dk, dv).
    """
    lib = _lib.load()
    _check3("q", q)
    for name, t in (("k", k), ("v", v), ("dout", dout)):
        _check3(name, t, q.dtype)
    bh, nq, h = q.shape
    nk = k.shape[1]
    group = _kv_group(bh, k)
    if k.shape != (bh // group, nk, h) or v.shape != k.shape or dout.shape != q.shape:
        raise ShapeError("q/k/v/dout do not conform")
    if lse.shape != (bh, nq) or delta.shape != (bh, nq):
        raise ShapeError("lse / delta must be [bh, nq]")
    if not (lse.is_contiguous() and delta.is_contiguous()):
        raise ShapeError("lse / delta must be contiguous")
    qi = q_index if q_index is not None else TokenIndex.contiguous(nq)
    ki = k_index if k_index is not None else TokenIndex.contiguous(nk)
    if qi.n != nq or ki.n != nk:
        raise ShapeError("index maps do not match the row counts")
    qi, ki = _pair_maps(qi, ki, causal, q.device)
    if dq_acc is None:
        dq_acc = torch.zeros((bh, nq, h), dtype=torch.float32, device=q.device)
    if accumulate_dkv and (dk is None or dv is None or dk.dtype != torch.float32):
        raise ShapeError("accumulate_dkv needs existing fp32 dk / dv")
    if dk is None:
        dk = torch.empty((bh, nk, h), dtype=dkv_dtype, device=q.device)
    if dv is None:
        dv = torch.empty((bh, nk, h), dtype=dkv_dtype, device=q.device)
    if dq_acc.dtype != torch.float32 or dq_acc.shape != (bh, nq, h) or dq_acc.stride(2) != 1:
        raise ShapeError("dq_acc must be fp32 [bh, nq, h] with unit stride along h")
    if dk.stride() != dv.stride() or dk.dtype != dv.dtype or dk.shape != (bh, nk, h):
        raise ShapeError("dk / dv must share shape, strides and dtype")
    a = _lib.TileBwdArgs()
    a.q, a.k, a.v, a.dout = q.data_ptr(), k.data_ptr(), v.data_ptr(), dout.data_ptr()
    a.lse, a.delta, a.dq_acc = lse.data_ptr(), delta.data_ptr(), dq_acc.data_ptr()
    a.dk, a.dv = dk.data_ptr(), dv.data_ptr()
    a.q_stride_bh, a.q_stride_row = q.stride(0), q.stride(1)
    a.k_stride_bh, a.k_stride_row = k.stride(0), k.stride(1)
    a.v_stride_bh, a.v_stride_row = v.stride(0), v.stride(1)
    a.do_stride_bh, a.do_stride_row = dout.stride(0), dout.stride(1)
    a.dq_stride_bh, a.dq_stride_row = dq_acc.stride(0), dq_acc.stride(1)
    a.dkv_stride_bh, a.dkv_stride_row = dk.stride(0), dk.stride(1)
    a.bh, a.nq, a.nk, a.h = bh, nq, nk, h
    a.causal = int(bool(causal))
    a.scale = float(scale)
    a.dkv_dtype = _dtype_code(dk.dtype)
    a.accumulate_dkv = int(bool(accumulate_dkv))
    a.q_map, a.k_map = qi.to_c(), ki.to_c()
    a.kv_group = group
    a.in_dtype = _dtype_code(q.dtype)
    _lib.check(lib.a2d_tile_bwd(a, _stream(q)), "a2d_tile_bwd")
    return dq_acc, dk, dv


def bwd_finalize(dq_acc: torch.Tensor, scale: float, out: torch.Tensor | None = None,
                 dtype: torch.dtype = torch.bfloat16) -> torch.Tensor:
    """dq = scale * dq_acc (numpy_backend.py:61)."""
    lib = _lib.load()
    bh, n, h = dq_acc.shape
    if out is None:
        out = torch.empty((bh, n, h), dtype=dtype, device=dq_acc.device)
    _lib.check(lib.a2d_bwd_finalize(dq_acc.data_ptr(), dq_acc.stride(0), dq_acc.stride(1),
                                    out.data_ptr(), _dtype_code(out.dtype), out.stride(0),
                                    out.stride(1), bh, n, h, float(scale), _stream(dq_acc)),
               "a2d_bwd_finalize")
    return out


def lse_merge(o_parts: torch.Tensor, lse_parts: torch.Tensor, *,
              out: torch.Tensor | None = None, lse_out: torch.Tensor | None = None,
              out_dtype: torch.dtype = torch.bfloat16):
    """k-way merge of partials: o_parts [k, rows, h] fp32, lse_parts [k, rows]
    -> (o [rows, h], lse [rows]).  attn_fix folded + finalize
    (attention.py:194-222)."""
    lib = _lib.load()
    if o_parts.dim() != 3 or lse_parts.dim() != 2:
        raise ShapeError("o_parts must be [k, rows, h] and lse_parts [k, rows]")
    kp, rows, h = o_parts.shape
    if lse_parts.shape != (kp, rows):
        raise ShapeError("lse_parts does not match o_parts")
    if o_parts.dtype != torch.float32 or lse_parts.dtype != torch.float32:
        raise ShapeError("partials must be fp32")
    if o_parts.stride(2) != 1 or lse_parts.stride(1) != 1:
        raise ShapeError("partials need unit inner stride")
    if out is None:
        out = torch.empty((rows, h), dtype=out_dtype, device=o_parts.device)
    if lse_out is None:
        lse_out = torch.empty((rows,), dtype=torch.float32, device=o_parts.device)
    _lib.check(lib.a2d_lse_merge(o_parts.data_ptr(), lse_parts.data_ptr(), kp,
                                 o_parts.stride(0), lse_parts.stride(0), rows, h,
                                 o_parts.stride(1), out.data_ptr(), _dtype_code(out.dtype),
                                 out.stride(0), lse_out.data_ptr(), _stream(o_parts)),
               "a2d_lse_merge")
    return out, lse_out


def selftest_umma(a: torch.Tensor, b: torch.Tensor, b_mn_major: bool) -> torch.Tensor:
    lib = _lib.load()
    n = b.shape[1] if b_mn_major else b.shape[0]
    d = torch.empty((128, n), dtype=torch.float32, device=a.device)
    _lib.check(lib.a2d_selftest_umma(a.data_ptr(), b.data_ptr(), d.data_ptr(), n,
                                     int(b_mn_major), _stream(a)), "a2d_selftest_umma")
    return d


def debug_poison(mode: int = 3, device=None) -> None:
    """Diagnostic: fill SMEM (bit 0) and TMEM (bit 1) of every SM with NaNs."""
    lib = _lib.load()
    dev = torch.device(device) if device is not None else torch.device("cuda")
    _lib.check(lib.a2d_debug_poison(int(mode), torch.cuda.current_stream(dev).cuda_stream),
               "a2d_debug_poison")
