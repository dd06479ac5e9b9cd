"""The CPU oracle (oracle/attn2d_oracle.py) pinned against the reference:
golden vectors produced by the unmodified reference package
(tests/golden/make_golden.py) and its known-answer tests."""

import itertools
from pathlib import Path

import numpy as np
import pytest

from oracle import attn2d_oracle as orc

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def tile():
    return np.load(GOLD / "tile_small.npz")


@pytest.mark.parametrize("tag", ["none", "causal"])
def test_flash_forward_matches_reference(tile, tag):
    g = {k[len(tag) + 1:]: tile[k] for k in tile.files if k.startswith(tag + "_")}
    m, n, d = orc.empty_partial(*g["q"].shape)
    orc.flash_forward(g["q"], g["k"], g["v"], g["q_idx"], g["k_idx"], tag == "causal", 1.0, 64,
                      m, n, d)
    assert np.allclose(m, g["m"], atol=1e-13, equal_nan=True)
    assert np.allclose(n, g["n"], atol=1e-13)
    assert np.allclose(d, g["d"], atol=1e-13)


@pytest.mark.parametrize("tag", ["none", "causal"])
@pytest.mark.parametrize("block", [1, 2, 5, 64])
def test_flash_forward_block_invariance(tile, tag, block):
    """test_kernels.py:112-122: the recurrence does not depend on the block."""
    g = {k[len(tag) + 1:]: tile[k] for k in tile.files if k.startswith(tag + "_")}
    m, n, d = orc.empty_partial(*g["q"].shape)
    orc.flash_forward(g["q"], g["k"], g["v"], g["q_idx"], g["k_idx"], tag == "causal", 1.0,
                      block, m, n, d)
    lse = orc.logsumexp(m, d)
    want = orc.logsumexp(g["m"], g["d"])
    assert np.allclose(lse, want, atol=1e-12, equal_nan=True)


@pytest.mark.parametrize("tag", ["none", "causal"])
def test_flash_backward_matches_reference(tile, tag):
    g = {k[len(tag) + 1:]: tile[k] for k in tile.files if k.startswith(tag + "_")}
    dq, dk, dv = (np.zeros_like(g[x]) for x in ("q", "k", "v"))
    orc.flash_backward(g["q"], g["k"], g["v"], g["o"], g["dout"], g["m"], g["d"], g["q_idx"],
                       g["k_idx"], tag == "causal", 1.0, dq, dk, dv)
    for got, key in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        assert np.abs(got - g[key]).max() < 1e-12


def test_known_answers(tile):
    """SPEC.md:114-116, :132-133 and test_attention.py:61-69, :147-157."""
    q = np.zeros((1, 1))
    assert np.allclose(orc.reference_attention(q, np.zeros((1, 1)), np.array([[3.0]])), [[3.0]])
    assert np.allclose(orc.reference_attention(np.zeros((2, 1)), np.zeros((2, 1)),
                                               np.array([[1.0], [3.0]])), [[2.0], [2.0]])
    assert np.allclose(orc.reference_attention(np.zeros((2, 1)), np.zeros((2, 1)),
                                               np.array([[1.0], [3.0]]), causal=True),
                       [[1.0], [2.0]])
    m, n, d = orc.empty_partial(1, 1)
    orc.flash_forward(np.zeros((1, 1)), np.zeros((2, 1)), np.array([[2.0], [4.0]]),
                      np.array([0]), np.array([0, 1]), False, 1.0, 1, m, n, d)
    assert (m[0], n[0, 0], d[0]) == (0.0, 6.0, 2.0)
    assert np.array_equal(m, tile["kat_tile_m"]) and np.array_equal(n, tile["kat_tile_n"])
    # masked row stays the empty partial
    m, n, d = orc.empty_partial(2, 2)
    orc.flash_forward(tile["masked_q"], tile["masked_k"], tile["masked_v"], np.array([0, 8]),
                      np.array([4, 5]), True, 1.0, 64, m, n, d)
    assert m[0] == -np.inf and d[0] == 0 and np.all(n[0] == 0)
    assert np.allclose(n, tile["masked_n"]) and np.allclose(d, tile["masked_d"])
    with pytest.raises(ZeroDivisionError):
        orc.finalize((m, n, d))


def test_index_subsets(tile):
    o, lse, _ = orc.tile_forward_full(tile["subset_q"], tile["subset_k"], tile["subset_v"],
                                      tile["subset_q_idx"], tile["subset_k_idx"], True, 1.0)
    assert np.abs(o - tile["subset_o"]).max() < 1e-13
    assert np.abs(lse - tile["subset_lse"]).max() < 1e-13


def test_attn_fix_known_answer_and_fold():
    g = np.load(GOLD / "merge_small.npz")
    m, n, d = orc.attn_fix((np.array([0.0]), np.array([[1.0]]), np.array([1.0])),
                           (np.array([0.0]), np.array([[3.0]]), np.array([1.0])))
    assert (m[0], n[0, 0], d[0]) == (g["kat_m"][0], g["kat_n"][0, 0], g["kat_d"][0]) == (0, 4, 2)
    parts = [(g[f"part{i}_m"], g[f"part{i}_n"], g[f"part{i}_d"]) for i in range(4)]
    # every grouping / order of the fold agrees (test_acceptance.py:137-175)
    for perm in itertools.permutations(range(4)):
        acc = parts[perm[0]]
        for i in perm[1:]:
            acc = orc.attn_fix(acc, parts[i])
        assert np.abs(orc.finalize(acc) - g["fold_o"]).max() < 1e-12
        assert np.abs(orc.logsumexp(acc[0], acc[2]) - g["fold_lse"]).max() < 1e-12
    # the LSE-form k-way merge (what the CUDA kernel computes) equals the fold
    o_parts, lse_parts = [], []
    for m_, n_, d_ in parts:
        live = d_ > 0
        o_parts.append(np.where(live[:, None], n_ / np.where(live, d_, 1)[:, None], 0.0))
        lse_parts.append(orc.logsumexp(m_, d_))
    o, lse = orc.lse_merge(o_parts, lse_parts)
    assert np.abs(o - g["fold_o"]).max() < 1e-12
    assert np.abs(lse - g["fold_lse"]).max() < 1e-12


def test_empty_partial_is_bitwise_identity():
    """test_attention.py:188-201."""
    rng = np.random.default_rng(50)
    q, k, v = rng.uniform(-1, 1, (4, 3)), rng.uniform(-1, 1, (5, 3)), rng.uniform(-1, 1, (5, 3))
    part = orc.empty_partial(4, 3)
    orc.flash_forward(q, k, v, np.arange(4), np.arange(5), False, 1.0, 64, *part)
    e = orc.empty_partial(4, 3)
    for merged in (orc.attn_fix(part, e), orc.attn_fix(e, part)):
        for a, b in zip(merged, part):
            assert np.array_equal(a, b)


def test_dense_gradient_finite_differences():
    """test_attention.py:260-289: central differences of the dense oracle."""
    rng = np.random.default_rng(7)
    q, k, v, do = (rng.uniform(-1, 1, (5, 3)) for _ in range(4))
    dq, dk, dv = orc.reference_attention_grad(q, k, v, do, causal=True, scale=0.7)
    eps = 1e-6
    f = lambda q_, k_, v_: float(np.sum(orc.reference_attention(q_, k_, v_, True, 0.7) * do))
    for arr, grad, which in ((q, dq, 0), (k, dk, 1), (v, dv, 2)):
        i, j = 3, 1
        plus, minus = [q.copy(), k.copy(), v.copy()], [q.copy(), k.copy(), v.copy()]
        plus[which][i, j] += eps
        minus[which][i, j] -= eps
        fd = (f(*plus) - f(*minus)) / (2 * eps)
        assert abs(fd - grad[i, j]) < 1e-6


@pytest.mark.parametrize("tag", ["n256_h64_causal", "n128_h128_causal"])
def test_oracle_on_gpu_parity_fixture(tag):
    """The fixtures the GPU tests use are the reference's outputs; the oracle
    reproduces them from the same bf16-rounded inputs."""
    g = np.load(GOLD / "gpu_parity.npz")
    n, h, causal, scale = g[f"{tag}_meta"]
    bits = lambda a: (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    q, k, v, do = (bits(g[f"{tag}_{x}"]) for x in ("q", "k", "v", "dout"))
    idx = np.arange(int(n))
    o, lse, (m, d) = orc.tile_forward_full(q, k, v, idx, idx, bool(causal), float(scale))
    assert np.abs(o - g[f"{tag}_o"]).max() < 1e-6
    assert np.abs(lse - g[f"{tag}_lse"]).max() < 1e-5
    dq, dk, dv = orc.tile_backward_full(q, k, v, o, do, m, d, idx, idx, bool(causal), float(scale))
    for got, key in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        assert np.abs(got - g[f"{tag}_{key}"]).max() < 1e-5
    assert int(g[f"{tag}_pairs"]) == orc.count_unmasked(idx, idx, bool(causal))


def test_layouts_and_counts():
    """layouts.py:53-65 and the causal work counts of test_strategies.py:279-309."""
    n, p = 8, 4
    counts = {}
    for r in range(2):
        for c in range(2):
            qi = orc.cyclic_indices(n, p, "row_gathered", r, c)
            ki = orc.cyclic_indices(n, p, "col_gathered", r, c)
            counts[(r, c)] = orc.count_unmasked(qi, ki, True)
    assert counts == {(0, 0): 10, (0, 1): 6, (1, 0): 10, (1, 1): 10}
    ring = [orc.count_unmasked(orc.ring_block_indices(n, p, rk), np.arange(n), True)
            for rk in range(p)]
    assert ring == [9, 9, 9, 9]
    assert orc.ring_block_indices(8, 4, 1).tolist() == [1, 6]
