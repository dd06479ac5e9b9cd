"""CPU-side checks of the C ABI and the host logic (no compute calls):
the shared library loads and exports every symbol include/attn2d_b200.h
declares, the ctypes structs match the C layout, and the layout / index-map
logic reproduces the reference's layouts."""

import ctypes
import re
import subprocess
import tempfile
from pathlib import Path

import numpy as np
import pytest

from oracle import attn2d_oracle as orc
from paper_2503_15758_b200 import _lib
from paper_2503_15758_b200.errors import ConfigError, ShapeError
from paper_2503_15758_b200.layouts import Grid2D, ring_block_indices, ring_index
from paper_2503_15758_b200.ops import TokenIndex

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "attn2d_b200.h"


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(a2d_\w+)\s*\(", HEADER.read_text(),
                              re.M))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name)
    assert lib.a2d_abi_version() == _lib.ABI_VERSION
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}\b", out), name


def test_ctypes_structs_match_c_layout():
    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "attn2d_b200.h"
int main(void) {
  printf("%zu %zu %zu\n", sizeof(a2d_index_map), sizeof(a2d_tile_fwd_args), sizeof(a2d_tile_bwd_args));
  printf("%zu %zu %zu %zu\n", offsetof(a2d_tile_fwd_args, q_map), offsetof(a2d_tile_fwd_args, k_map),
         offsetof(a2d_tile_bwd_args, q_map), offsetof(a2d_tile_bwd_args, dkv_dtype));
  printf("%zu %zu\n", offsetof(a2d_index_map, base), offsetof(a2d_index_map, idx));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = Path(d) / "s.c"
        c.write_text(src)
        exe = Path(d) / "s"
        subprocess.run(["gcc", "-I", str(ROOT / "include"), str(c), "-o", str(exe)], check=True)
        vals = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                                check=True).stdout.split()]
    F, B, M = _lib.TileFwdArgs, _lib.TileBwdArgs, _lib.IndexMap
    assert vals == [ctypes.sizeof(M), ctypes.sizeof(F), ctypes.sizeof(B),
                    F.q_map.offset, F.k_map.offset, B.q_map.offset, B.dkv_dtype.offset,
                    M.base.offset, M.idx.offset]


@pytest.mark.parametrize("p", [1, 4, 9, 16])
def test_square_grid_reproduces_reference_layouts(p):
    g = Grid2D.square(p)
    n = 4 * p
    for r, c in g.coords():
        assert np.array_equal(g.owned(n, r, c), orc.cyclic_indices(n, p, "column_major", r, c))
        assert np.array_equal(g.kv_owned(n, r, c), orc.cyclic_indices(n, p, "row_major", r, c))
        assert np.array_equal(np.sort(g.q_gathered(n, r).host()),
                              orc.cyclic_indices(n, p, "row_gathered", r, c))
        assert np.array_equal(np.sort(g.k_gathered(n, c).host()),
                              orc.cyclic_indices(n, p, "col_gathered", r, c))
        # the permutation is the reference's mirror transpose (r, c) <-> (c, r)
        assert g.kv_dest(r, c) == g.rank(c, r) and g.kv_src(r, c) == g.rank(c, r)


@pytest.mark.parametrize("pr,pc", [(1, 8), (2, 4), (4, 2), (8, 1), (2, 1), (1, 2)])
def test_rect_grid_gathers_are_consistent(pr, pc):
    g = Grid2D(pr, pc)
    n = 8 * g.p
    for r, c in g.coords():
        # what the row members own, concatenated in gather order, is q_gathered
        qg = np.concatenate([g.owned(n, r, cc) for cc in range(pc)])
        assert np.array_equal(qg, g.q_gathered(n, r).host())
        # after the permutation, (r, c) holds the row-major residue it needs
        src = g.coord(g.kv_src(r, c))
        assert np.array_equal(g.owned(n, *src), g.kv_owned(n, r, c))
        kg = np.concatenate([g.kv_owned(n, rr, c) for rr in range(pr)])
        assert np.array_equal(kg, g.k_gathered(n, c).host())
        assert g.kv_src(*g.coord(g.kv_dest(r, c))) == g.rank(r, c)
    # every token is owned exactly once
    allq = np.sort(np.concatenate([g.owned(n, r, c) for r, c in g.coords()]))
    assert np.array_equal(allq, np.arange(n))


def test_ring_layout_matches_reference():
    for n, p in ((8, 4), (16, 4), (32, 8), (48, 4)):
        for rk in range(p):
            assert np.array_equal(ring_block_indices(n, p, rk), orc.ring_block_indices(n, p, rk))
            assert np.array_equal(ring_index(n, p, rk).host(), orc.ring_block_indices(n, p, rk))
    with pytest.raises(ConfigError):
        ring_block_indices(12, 4, 0)


def test_token_index_detection():
    assert not TokenIndex.from_indices(np.arange(5, 105, 3)).is_array
    blk = np.concatenate([np.arange(7, 7 + 8 * 256, 8), np.arange(3, 3 + 8 * 256, 8)])
    ti = TokenIndex.from_indices(blk)
    assert not ti.is_array and ti.bases == (7, 3) and ti.stride == 8 and ti.rows_per_block == 256
    assert np.array_equal(ti.host(), blk)
    m = ti.to_c()
    assert m.mode == _lib.IDX_AFFINE and m.nblocks == 2 and m.base[1] == 3


def test_error_taxonomy_mapping():
    class FakeLib:
        def a2d_last_error(self):
            return b"boom"
    _lib._LIB, saved = FakeLib(), _lib._LIB
    try:
        with pytest.raises(ShapeError):
            _lib.check(_lib.A2D_EINVAL, "x")
        with pytest.raises(_lib.UnsupportedError):
            _lib.check(_lib.A2D_EUNSUPPORTED, "x")
        with pytest.raises(RuntimeError):
            _lib.check(_lib.A2D_ECUDA, "x")
    finally:
        _lib._LIB = saved


def test_no_cpu_fallback():
    """The product path refuses to run without the CUDA extension or on host
    tensors: there is no CPU fallback to silently take over."""
    import torch
    from paper_2503_15758_b200 import ops
    with pytest.raises(RuntimeError):
        _lib.load("/nonexistent/libattn2d_b200.so")
    q = torch.zeros((1, 128, 64), dtype=torch.bfloat16)
    with pytest.raises(ShapeError):
        ops.tile_forward(q, q, q, causal=True, scale=0.125)


def test_abi_argument_validation_without_a_gpu():
    """Invalid calls are rejected by the C ABI before any CUDA work, with the
    documented return codes (include/attn2d_b200.h)."""
    lib = _lib.load()
    a = _lib.TileFwdArgs()
    a.q = a.k = a.v = a.o = a.lse = 16  # never dereferenced: validation fails first
    a.bh, a.nq, a.nk, a.causal, a.scale, a.o_dtype = 2, 128, 128, 1, 0.125, _lib.BF16
    for m in (a.q_map, a.k_map):
        m.mode, m.nblocks, m.rows_per_block, m.stride = _lib.IDX_AFFINE, 1, 128, 1
    a.h = 100                                   # not a multiple of 8
    assert lib.a2d_tile_fwd(a, None) == _lib.A2D_EUNSUPPORTED
    a.h = 136                                   # wider than the tiles
    assert lib.a2d_tile_fwd(a, None) == _lib.A2D_EUNSUPPORTED
    a.h, a.kv_group = 64, 3                     # 3 does not divide bh = 2
    assert lib.a2d_tile_fwd(a, None) == _lib.A2D_EINVAL
    a.kv_group, a.nq = 1, -1
    assert lib.a2d_tile_fwd(a, None) == _lib.A2D_EINVAL
    assert b"negative" in lib.a2d_last_error()


def test_abi_empty_calls_succeed_with_null_buffers():
    """Zero heads or zero rows is a valid call that touches no memory: empty
    torch tensors carry null data pointers, so the null checks come after
    the emptiness checks (no CUDA work, so this runs without a GPU)."""
    lib = _lib.load()
    a = _lib.TileFwdArgs()
    a.nq, a.nk, a.h, a.causal, a.scale, a.o_dtype = 128, 128, 64, 1, 0.125, _lib.F32
    for m in (a.q_map, a.k_map):
        m.mode, m.nblocks, m.rows_per_block, m.stride = _lib.IDX_AFFINE, 1, 128, 1
    a.bh = 0
    assert lib.a2d_tile_fwd(a, None) == _lib.A2D_OK
    a.bh, a.nq, a.q_map.rows_per_block = 2, 0, 0
    assert lib.a2d_tile_fwd(a, None) == _lib.A2D_OK
    assert lib.a2d_bwd_preprocess(None, None, None, 0, 0, 0, 0, 0, 128, 64, _lib.BF16,
                                  None) == _lib.A2D_OK
    assert lib.a2d_bwd_finalize(None, 0, 0, None, _lib.F32, 0, 0, 2, 0, 64, 1.0, None) == _lib.A2D_OK
    assert lib.a2d_lse_merge(None, None, 2, 0, 0, 0, 64, 64, None, _lib.F32, 64, None,
                             None) == _lib.A2D_OK
    assert lib.a2d_bwd_preprocess(None, None, None, 0, 0, 0, 0, -1, 128, 64, _lib.F16,
                                  None) == _lib.A2D_EINVAL
    # 16-bit inputs only (0, the v3 reserved value, reads as bf16)
    assert lib.a2d_bwd_preprocess(None, None, None, 0, 0, 0, 0, 1, 128, 64, 3,
                                  None) == _lib.A2D_EUNSUPPORTED
