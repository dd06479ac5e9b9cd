"""ctypes binding of libattn2d_b200.so (include/attn2d_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` (or
`make -C paper_2503_15758_b200/csrc`).  There is no fallback: importing the
compute path without the library raises immediately.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_float, c_int32, c_int64, c_void_p
from pathlib import Path

from .errors import ShapeError, UnsupportedError

LIB_PATH = Path(os.environ.get("A2D_LIB_PATH") or
                Path(__file__).resolve().parent / "libattn2d_b200.so")
ABI_VERSION = 4
MAX_BLOCKS = 16

A2D_OK, A2D_EINVAL, A2D_EUNSUPPORTED, A2D_ECUDA = 0, 1, 2, 3
IDX_AFFINE, IDX_ARRAY = 0, 1
F32, BF16, F16 = 0, 1, 2

# every symbol include/attn2d_b200.h declares
EXPORTS = ("a2d_tile_fwd", "a2d_bwd_preprocess", "a2d_tile_bwd", "a2d_bwd_finalize",
           "a2d_lse_merge", "a2d_selftest_umma", "a2d_bench_umma", "a2d_debug_poison", "a2d_abi_version", "a2d_last_error",
           "a2d_num_sms")


class IndexMap(ctypes.Structure):
    _fields_ = [("mode", c_int32), ("nblocks", c_int32), ("rows_per_block", c_int32),
                ("reserved", c_int32), ("stride", c_int64), ("base", c_int64 * MAX_BLOCKS),
                ("idx", c_void_p)]


class TileFwdArgs(ctypes.Structure):
    _fields_ = [("q", c_void_p), ("k", c_void_p), ("v", c_void_p), ("o", c_void_p),
                ("lse", c_void_p),
                ("q_stride_bh", c_int64), ("q_stride_row", c_int64),
                ("k_stride_bh", c_int64), ("k_stride_row", c_int64),
                ("v_stride_bh", c_int64), ("v_stride_row", c_int64),
                ("o_stride_bh", c_int64), ("o_stride_row", c_int64),
                ("bh", c_int32), ("nq", c_int32), ("nk", c_int32), ("h", c_int32),
                ("causal", c_int32), ("scale", c_float), ("o_dtype", c_int32),
                ("accumulate", c_int32), ("q_map", IndexMap), ("k_map", IndexMap),
                ("kv_group", c_int32), ("in_dtype", c_int32)]


class TileBwdArgs(ctypes.Structure):
    _fields_ = [("q", c_void_p), ("k", c_void_p), ("v", c_void_p), ("dout", c_void_p),
                ("lse", c_void_p), ("delta", c_void_p), ("dq_acc", c_void_p),
                ("dk", c_void_p), ("dv", c_void_p),
                ("q_stride_bh", c_int64), ("q_stride_row", c_int64),
                ("k_stride_bh", c_int64), ("k_stride_row", c_int64),
                ("v_stride_bh", c_int64), ("v_stride_row", c_int64),
                ("do_stride_bh", c_int64), ("do_stride_row", c_int64),
                ("dq_stride_bh", c_int64), ("dq_stride_row", c_int64),
                ("dkv_stride_bh", c_int64), ("dkv_stride_row", c_int64),
                ("bh", c_int32), ("nq", c_int32), ("nk", c_int32), ("h", c_int32),
                ("causal", c_int32), ("scale", c_float), ("dkv_dtype", c_int32),
                ("accumulate_dkv", c_int32), ("q_map", IndexMap), ("k_map", IndexMap),
                ("kv_group", c_int32), ("in_dtype", c_int32)]


_LIB = None


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library; raise if it is missing."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} not found: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = ctypes.CDLL(str(p))
    lib.a2d_tile_fwd.argtypes = [ctypes.POINTER(TileFwdArgs), c_void_p]
    lib.a2d_tile_bwd.argtypes = [ctypes.POINTER(TileBwdArgs), c_void_p]
    lib.a2d_bwd_preprocess.argtypes = [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64,
                                       c_int64, c_int32, c_int32, c_int32, c_int32, c_void_p]
    lib.a2d_bwd_finalize.argtypes = [c_void_p, c_int64, c_int64, c_void_p, c_int32, c_int64,
                                     c_int64, c_int32, c_int32, c_int32, c_float, c_void_p]
    lib.a2d_lse_merge.argtypes = [c_void_p, c_void_p, c_int32, c_int64, c_int64, c_int64,
                                  c_int32, c_int64, c_void_p, c_int32, c_int64, c_void_p,
                                  c_void_p]
    lib.a2d_bench_umma.argtypes = [c_int32, c_int32, c_void_p, c_int32, c_void_p]
    lib.a2d_debug_poison.argtypes = [c_int32, c_void_p]
    lib.a2d_selftest_umma.argtypes = [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p]
    lib.a2d_last_error.restype = ctypes.c_char_p
    for name in EXPORTS:
        getattr(lib, name)
    if lib.a2d_abi_version() != ABI_VERSION:
        raise RuntimeError(f"ABI mismatch: library {lib.a2d_abi_version()} != {ABI_VERSION}")
    if path is None:
        _LIB = lib
    return lib


def check(rc: int, what: str) -> None:
    """Map ABI return codes onto the reference's exception taxonomy
    (errors.py:4-21)."""
    if rc == A2D_OK:
        return
    msg = f"{what}: {_LIB.a2d_last_error().decode(errors='replace') if _LIB else rc}"
    if rc == A2D_EINVAL:
        raise ShapeError(msg)
    if rc == A2D_EUNSUPPORTED:
        raise UnsupportedError(msg)
    raise RuntimeError(msg)
