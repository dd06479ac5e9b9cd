"""The B200 path as a drop-in for the reference's attention entry points.

Two layers of evidence (VERDICT r1 "prove the drop-in"):

* Fixture tests (no reference needed at run time): the reference's own
  attention-API test vectors, computed by the UNMODIFIED reference on
  bf16-rounded inputs (`tests/golden/make_golden.py::dropin_cases` ->
  `dropin.npz`), are fed through this package's mirrors of that API —
  `kernels.flash_forward / flash_backward` (the in-place (m, nacc, d)
  contract, reference kernels/__init__.py:70-92) and
  `attention.flash_attn_forward / flash_attn_backward / attn_fix / finalize /
  PartialAttn` (attention.py:75-257).
* Live-reference tests: the reference package itself (pip-installed into
  `baseline/_ref`) gets this package's kernel module
  registered as one more entry of its backend table
  (`attn2d.kernels._BACKENDS["b200"]`, exactly as INTEGRATION.md §2 shows),
  and the reference's OWN code — `flash_attn_forward/backward`, `finalize`,
  `run_forward/run_backward` for attn2d_no, attn2d_o and ring on its
  simulated grid — runs on the sm_100a kernels, compared with the same calls
  on its numpy backend.

Tolerance (SURVEY.md §8c, bf16 P / fp32 accumulation vs fp64): rel-Fro
<= 1e-2 and max-abs <= 2e-2 * max|ref| on O, dQ, dK, dV; LSE max-abs <= 1e-3.
Known answers with exactly representable values must match exactly.
"""

from __future__ import annotations

import inspect
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden" / "dropin.npz"
REF = ROOT / "baseline" / "_ref"
REL_TOL, ABS_FRAC, LSE_TOL = 1e-2, 2e-2, 1e-3


def _close(got, want, what=""):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    if want.size == 0:
        return
    err = np.abs(got - want)
    scale = max(float(np.abs(want).max()), 1e-30)
    rel = float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))
    assert rel <= REL_TOL and float(err.max()) <= ABS_FRAC * scale, \
        f"{what}: rel-Fro {rel:.3e}, max-abs {float(err.max()):.3e} (|ref| max {scale:.3e})"


def _lse_close(got, want, what=""):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), fin), f"{what}: empty rows differ"
    if fin.any():
        err = float(np.abs(got[fin] - want[fin]).max())
        assert err <= LSE_TOL, f"{what}: LSE max-abs {err:.3e}"


def _np(t):
    return t.detach().double().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.fixture(scope="module")
def b200():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_15758_b200 import attention, kernels
    return kernels, attention


# --------------------------------------------------------------------------
# fixture tests: this package's mirrors of the reference API
# --------------------------------------------------------------------------

def _run_kernel_forward(kernels, q, k, v, qi, ki, causal, block=64, state=None):
    m, nacc, d = state if state is not None else (np.full(q.shape[0], -np.inf),
                                                  np.zeros_like(q), np.zeros(q.shape[0]))
    kernels.flash_forward(q, k, v, qi, ki, causal, 1.0, block, m, nacc, d)
    return m, nacc, d


def _observables(m, nacc, d):
    """(O, LSE) of a (m, n, d) triple: the reference's finalize and
    logsumexp (attention.py:103-107, 217-222)."""
    live = d > 0
    o = np.zeros_like(nacc)
    o[live] = nacc[live] / d[live, None]
    lse = np.where(live, m + np.log(np.where(live, d, 1.0)), -np.inf)
    return o, lse


@pytest.mark.gpu
def test_known_answer_tile(b200):
    """q=[0], k=[0,1], v=[[2],[4]], zero Q/K -> (M, N, D) =
    (0, [[6]], 2), i.e. O = 3 and LSE = log 2; the kernels keep the unique
    form (LSE, O, 1) of the same partial; fully masked -> (-inf, 0, 0).
    SPEC.md:114-116 answers hold to fp32 rounding: with a non-zero score the
    kernel's fused scale-and-subtract leaves 2^(x - m) one ulp off 1 in the
    fp32 denominator (a 1e-7 relative effect)."""
    kernels, attention = b200
    m, nacc, d = _run_kernel_forward(kernels, np.zeros((1, 1)), np.zeros((2, 1)),
                                     np.array([[2.0], [4.0]]), np.array([0]), np.array([0, 1]),
                                     False, block=1)
    o, lse = _observables(m, nacc, d)
    assert o[0, 0] == 3.0
    assert abs(lse[0] - np.log(2.0)) < 1e-6
    m, nacc, d = _run_kernel_forward(kernels, np.zeros((1, 1)), np.zeros((1, 1)),
                                     np.array([[5.0]]), np.array([0]), np.array([1]), True)
    assert m[0] == -np.inf and d[0] == 0.0 and nacc[0, 0] == 0.0
    # SPEC.md:114-116 through the streaming wrapper: one key, equal scores, causal
    sh = attention.TokenShard
    one = attention.finalize(attention.flash_attn_forward(
        sh(np.array([[1.0]]), [0]), sh(np.array([[7.0]]), [0]), sh(np.array([[3.0]]), [0])))
    assert abs(_np(one)[0, 0] - 3.0) < 3e-6
    z, v = np.zeros((2, 1)), np.array([[1.0], [3.0]])
    eq = attention.finalize(attention.flash_attn_forward(sh(z, [0, 1]), sh(z, [0, 1]),
                                                         sh(v, [0, 1])))
    assert np.array_equal(_np(eq), [[2.0], [2.0]])  # zero scores: exact
    ca = attention.finalize(attention.flash_attn_forward(sh(z, [0, 1]), sh(z, [0, 1]),
                                                         sh(v, [0, 1]),
                                                         attention.MaskSpec.causal()))
    assert np.array_equal(_np(ca), [[1.0], [2.0]])


@pytest.mark.gpu
@pytest.mark.parametrize("mask", ["none", "causal"])
@pytest.mark.parametrize("block", [1, 3, 64])
def test_flash_attn_forward_matches_reference(b200, gold, mask, block):
    """test_attention.py:123-130 vectors through attention.flash_attn_forward."""
    _, attention = b200
    q, k, v = (gold[f"fw_{x}"] for x in "qkv")
    idx = np.arange(7)
    sh = attention.TokenShard
    ms = attention.MaskSpec.causal() if mask == "causal" else attention.MaskSpec.none()
    part = attention.flash_attn_forward(sh(q, idx), sh(k, idx), sh(v, idx), ms, block=block)
    _close(_np(attention.finalize(part)), gold[f"fw_{mask}_b{block}_o"], "O")
    _lse_close(_np(part.logsumexp), gold[f"fw_{mask}_b{block}_lse"], "LSE")


@pytest.mark.gpu
def test_index_subsets_and_masked_rows(b200, gold):
    """Global indices drive causal masking (test_attention.py:136-145); a row
    that sees no key comes back empty, and finalize raises
    FullyMaskedRowError (:147-157)."""
    _, attention = b200
    from paper_2503_15758_b200.errors import FullyMaskedRowError
    sh = attention.TokenShard
    part = attention.flash_attn_forward(sh(gold["sub_q"], gold["sub_qi"]),
                                        sh(gold["sub_k"], gold["sub_ki"]),
                                        sh(gold["sub_v"], gold["sub_ki"]),
                                        attention.MaskSpec.causal())
    _close(_np(attention.finalize(part)), gold["sub_o"], "O")
    _lse_close(_np(part.logsumexp), gold["sub_lse"], "LSE")
    part = attention.flash_attn_forward(sh(gold["msk_q"], [0, 8]), sh(gold["msk_k"], [4, 5]),
                                        sh(gold["msk_v"], [4, 5]), attention.MaskSpec.causal())
    assert _np(part.m)[0] == -np.inf and _np(part.d)[0] == 0.0
    assert np.all(_np(part.n)[0] == 0.0) and _np(part.d)[1] > 0
    _lse_close(_np(part.logsumexp), gold["msk_lse"], "LSE")
    _close(_np(part.o)[1], gold["msk_o1"], "O row 1")
    with pytest.raises(FullyMaskedRowError):
        attention.finalize(part)


@pytest.mark.gpu
def test_streaming_continuation_in_place(b200, gold):
    """Two kernels.flash_forward calls over split key ranges continue the
    caller's (m, nacc, d) in place and equal one call
    (test_kernels.py:124-137)."""
    kernels, _ = b200
    q, k, v, qi, ki = (gold[f"cont_{x}"] for x in ("q", "k", "v", "qi", "ki"))
    q, k, v = (x.astype(np.float64) for x in (q, k, v))
    whole = _observables(*_run_kernel_forward(kernels, q, k, v, qi, ki, False))
    state = (np.full(q.shape[0], -np.inf), np.zeros_like(q), np.zeros(q.shape[0]))
    _run_kernel_forward(kernels, q, k[:4], v[:4], qi, ki[:4], False, state=state)
    _run_kernel_forward(kernels, q, k[4:], v[4:], qi, ki[4:], False, state=state)
    split = _observables(*state)
    for got, w, ref, what in zip(split, whole, (gold["cont_o"], gold["cont_lse"]), ("O", "LSE")):
        if what == "O":
            _close(got, ref, "continued O")
            _close(w, ref, "whole O")
        else:
            _lse_close(got, ref, "continued LSE")
            _lse_close(w, ref, "whole LSE")


@pytest.mark.gpu
@pytest.mark.parametrize("mask", ["none", "causal"])
def test_flash_attn_backward_and_key_subset_partial_sums(b200, gold, mask):
    """flash_attn_backward over all keys (test_attention.py:289-300) and over
    key subsets with the global statistics: dq adds up, dk/dv slices
    concatenate (:302-328)."""
    _, attention = b200
    g = {x: gold[f"bw_{mask}_{x}"].astype(np.float64)
         for x in ("q", "k", "v", "do", "o", "lse", "dq", "dk", "dv")}
    ms = attention.MaskSpec.causal() if mask == "causal" else attention.MaskSpec.none()
    sh = attention.TokenShard
    n = g["q"].shape[0]
    idx = np.arange(n)
    part = attention.flash_attn_forward(sh(g["q"], idx), sh(g["k"], idx), sh(g["v"], idx), ms)
    o = attention.finalize(part)
    _close(_np(o), g["o"], "O")
    full = attention.flash_attn_backward(sh(g["q"], idx), sh(g["k"], idx), sh(g["v"], idx), o,
                                         g["do"], part.m, part.d, ms)
    for got, name in zip(full, ("dq", "dk", "dv")):
        _close(_np(got), g[name], name)
    dq_sum = np.zeros_like(g["q"])
    dk_got, dv_got = np.zeros_like(g["k"]), np.zeros_like(g["v"])
    for rows in (np.array([0, 2, 5]), np.array([1, 3]), np.array([4])):
        dq_i, dk_i, dv_i = attention.flash_attn_backward(
            sh(g["q"], idx), sh(g["k"][rows], rows), sh(g["v"][rows], rows), o, g["do"],
            part.m, part.d, ms)
        dq_sum += _np(dq_i)
        dk_got[rows] = _np(dk_i)
        dv_got[rows] = _np(dv_i)
    _close(dq_sum, g["dq"], "sum of dq partials")
    _close(dk_got, g["dk"], "dk slices")
    _close(dv_got, g["dv"], "dv slices")


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["mid_h64_causal", "mid_h128_none"])
def test_kernel_module_mid_size(b200, gold, tag):
    """kernels.flash_forward / flash_backward (reference signature, numpy
    in, caller-owned outputs accumulated in place) at h = 64 / 128 against
    the reference's numpy kernels on the same bf16 values."""
    kernels, _ = b200
    g = {x: gold[f"{tag}_{x}"].astype(np.float64)
         for x in ("q", "k", "v", "do", "o", "lse", "dq", "dk", "dv")}
    n, h, causal, sc = gold[f"{tag}_meta"]
    n, causal = int(n), bool(causal)
    idx = np.arange(n)
    m, nacc, d = np.full(n, -np.inf), np.zeros_like(g["q"]), np.zeros(n)
    kernels.flash_forward(g["q"], g["k"], g["v"], idx, idx, causal, float(sc), 64, m, nacc, d)
    o, lse = _observables(m, nacc, d)
    _close(o, g["o"], "O")
    _lse_close(lse, g["lse"], "LSE")
    # accumulate into non-zero caller buffers: the contract adds
    base = np.random.default_rng(0).uniform(-1, 1, (3,) + g["q"].shape)
    dq, dk, dv = base[0].copy(), base[1].copy(), base[2].copy()
    kernels.flash_backward(g["q"], g["k"], g["v"], g["o"], g["do"], m, d, idx, idx, causal,
                           float(sc), dq, dk, dv)
    for got, b, name in zip((dq, dk, dv), base, ("dq", "dk", "dv")):
        _close(got - b, g[name], name)


@pytest.mark.gpu
def test_partial_attn_algebra(b200, gold):
    """PartialAttn / attn_fix / finalize on the device: the empty partial is
    the identity, the merge is commutative, and folding key-subset partials
    equals one call (test_attention.py:188-244)."""
    _, attention = b200
    sh = attention.TokenShard
    q, k, v = (gold[f"fw_{x}"].astype(np.float64) for x in "qkv")
    idx = np.arange(7)
    whole = attention.flash_attn_forward(sh(q, idx), sh(k, idx), sh(v, idx))
    a = attention.flash_attn_forward(sh(q, idx), sh(k[:3], idx[:3]), sh(v[:3], idx[:3]))
    b = attention.flash_attn_forward(sh(q, idx), sh(k[3:], idx[3:]), sh(v[3:], idx[3:]))
    e = attention.PartialAttn.empty(7, v.shape[1])
    for merged in (attention.attn_fix(a, e), attention.attn_fix(e, a)):
        assert torch.equal(merged.lse, a.lse) and torch.equal(merged.o, a.o)
    ab, ba = attention.attn_fix(a, b), attention.attn_fix(b, a)
    assert torch.equal(ab.lse, ba.lse) and torch.equal(ab.o, ba.o)
    _close(_np(attention.finalize(ab)), _np(attention.finalize(whole)), "folded O")
    lse = np.logaddexp(_np(a.logsumexp), _np(b.logsumexp))
    assert np.abs(_np(ab.logsumexp) - lse).max() < 1e-5
    ee = attention.attn_fix(e, e)
    assert bool(torch.isneginf(ee.lse).all()) and bool((ee.d == 0).all())
    with pytest.raises(attention.ShapeError if hasattr(attention, "ShapeError") else Exception):
        attention.attn_fix(attention.PartialAttn.empty(2, 2), attention.PartialAttn.empty(3, 2))


@pytest.mark.gpu
def test_backward_rejects_empty_statistics(b200):
    """test_attention.py:330-334: d == 0 rows are FullyMaskedRowError."""
    _, attention = b200
    from paper_2503_15758_b200.errors import FullyMaskedRowError
    q = attention.TokenShard(np.zeros((2, 2)), [0, 1])
    with pytest.raises(FullyMaskedRowError):
        attention.flash_attn_backward(q, q, q, np.zeros((2, 2)), np.zeros((2, 2)),
                                      np.full(2, -np.inf), np.zeros(2))


@pytest.mark.gpu
def test_backward_value_head_dim_may_differ(b200):
    """Only q and k must share a head dim (attention.py:237-246): dq/dk keep
    q's width, dv v's."""
    _, attention = b200
    rng = np.random.default_rng(5)
    q, k, v, do = rng.uniform(-1, 1, (9, 16)), rng.uniform(-1, 1, (9, 16)), \
        rng.uniform(-1, 1, (9, 8)), rng.uniform(-1, 1, (9, 8))
    sh = attention.TokenShard
    idx = np.arange(9)
    part = attention.flash_attn_forward(sh(q, idx), sh(k, idx), sh(v, idx))
    o = attention.finalize(part)
    dq, dk, dv = attention.flash_attn_backward(sh(q, idx), sh(k, idx), sh(v, idx), o, do,
                                               part.m, part.d)
    assert tuple(dq.shape) == (9, 16) and tuple(dk.shape) == (9, 16) and tuple(dv.shape) == (9, 8)
    p = torch.softmax(torch.tensor(q) @ torch.tensor(k).T, -1)
    want_dv = (p.T @ torch.tensor(do)).numpy()
    _close(_np(dv), want_dv, "dv")


# --------------------------------------------------------------------------
# live reference: the b200 module registered in the reference's kernel table
# --------------------------------------------------------------------------

def _import_reference():
    if not (REF / "attn2d").is_dir():
        pytest.skip("reference not installed in baseline/_ref (BASELINE.md §4)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/a2d_numba_cache")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import attn2d.attention as ref_attention
    import attn2d.kernels as ref_kernels
    import attn2d.strategies as ref_strategies
    return ref_kernels, ref_attention, ref_strategies


@pytest.fixture(scope="module")
def reference():
    return _import_reference()


def test_kernel_module_matches_reference_signatures(reference):
    """The drop-in module exposes the reference kernel table's functions with
    the same parameter names and order (kernels/__init__.py:60-92), and the
    table accepts it as a backend."""
    ref_kernels, _, _ = reference
    from paper_2503_15758_b200 import kernels
    for name in ("flash_forward", "flash_backward", "matmul", "matmul_t", "use_backend",
                 "backend_name", "available_backends"):
        want = list(inspect.signature(getattr(ref_kernels, name)).parameters)
        got = list(inspect.signature(getattr(kernels, name)).parameters)
        assert got == want, (name, got, want)
    prev = ref_kernels.backend_name()
    ref_kernels._BACKENDS["b200"] = kernels
    try:
        assert ref_kernels.use_backend("b200") == "b200"
        assert "b200" in ref_kernels.available_backends()
    finally:
        ref_kernels.use_backend(prev)
        del ref_kernels._BACKENDS["b200"]


@pytest.fixture
def on_b200(reference):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ref_kernels, _, _ = reference
    from paper_2503_15758_b200 import kernels
    prev = ref_kernels.backend_name()
    ref_kernels._BACKENDS["b200"] = kernels

    def run(fn, backend):
        ref_kernels.use_backend(backend)
        try:
            return fn()
        finally:
            ref_kernels.use_backend(prev)

    yield run
    del ref_kernels._BACKENDS["b200"]


def _bf16(a):
    return torch.tensor(a, dtype=torch.float64).to(torch.bfloat16).double().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("causal", [False, True])
def test_reference_attention_api_runs_on_b200(reference, on_b200, causal):
    """The reference's flash_attn_forward / finalize / flash_attn_backward
    (attention.py:168-257), backend b200 vs backend numpy, same bf16 values;
    plus the SPEC known answers through its dense oracle and streaming path."""
    _, ra, _ = reference
    rng = np.random.default_rng(9)
    n, h = 200, 64
    q, k, v, do = (_bf16(rng.uniform(-1, 1, (n, h))) for _ in range(4))
    qi = np.arange(n) * 2 + 1           # index subsets: odd queries, all keys
    ki = np.arange(2 * n)[: n]
    mask = ra.MaskSpec.causal() if causal else ra.MaskSpec.none()
    sc = h ** -0.5

    def go():
        part = ra.flash_attn_forward(ra.TokenShard(q, qi), ra.TokenShard(k, ki),
                                     ra.TokenShard(v, ki), mask, sc, 64)
        o = ra.finalize(part)
        grads = ra.flash_attn_backward(ra.TokenShard(q, qi), ra.TokenShard(k, ki),
                                       ra.TokenShard(v, ki), o, do, part.m, part.d, mask, sc)
        return o, part.logsumexp, grads

    o_b, lse_b, g_b = on_b200(go, "b200")
    o_n, lse_n, g_n = on_b200(go, "numpy")
    _close(o_b, o_n, "O")
    _lse_close(lse_b, lse_n, "LSE")
    for a, b, name in zip(g_b, g_n, ("dq", "dk", "dv")):
        _close(a, b, name)

    def kat():
        sh = ra.TokenShard
        p = ra.flash_attn_forward(sh(np.zeros((1, 1)), [0]), sh(np.zeros((2, 1)), [0, 1]),
                                  sh(np.array([[2.0], [4.0]]), [0, 1]), ra.MaskSpec.none(), 1.0, 1)
        e = ra.flash_attn_forward(sh(np.zeros((1, 1)), [0]), sh(np.zeros((1, 1)), [1]),
                                  sh(np.array([[2.0]]), [1]), ra.MaskSpec.causal())
        return ra.finalize(p), p.logsumexp, e

    o, lse, e = on_b200(kat, "b200")
    assert o[0, 0] == 3.0 and abs(lse[0] - np.log(2.0)) < 1e-6
    assert e.m[0] == -np.inf and e.d[0] == 0.0 and e.n[0, 0] == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["attn2d_no", "attn2d_o", "ring"])
@pytest.mark.parametrize("p", [1, 4])
@pytest.mark.parametrize("causal", [False, True])
def test_reference_strategies_run_on_b200(reference, on_b200, gold, name, p, causal):
    """The reference's run_forward / run_backward (strategies/__init__.py:40-46)
    on its simulated p-processor grid with every tile call on the sm_100a
    kernels, against the reference's numpy-backend results on the same bf16
    inputs (the dropin.npz fixtures)."""
    _, ra, rs = reference
    n, h = 64, 8
    q, k, v, do = (x.astype(np.float64) for x in gold[f"st_in_p{p}"])
    mask = ra.MaskKind.CAUSAL if causal else ra.MaskKind.NONE
    cfg = rs.DistAttnConfig(n=n, h=h, p=p, mask=mask, scale=h ** -0.5)

    def go():
        fwd = rs.run_forward(name, cfg, q, k, v)
        bwd = rs.run_backward(name, cfg, fwd.saved, do)
        return fwd.o, bwd.dq, bwd.dk, bwd.dv

    got = on_b200(go, "b200")
    tag = f"st_{name}_p{p}_{'causal' if causal else 'none'}"
    for a, what in zip(got, ("o", "dq", "dk", "dv")):
        _close(a, gold[f"{tag}_{what}"], f"{name} p={p} {what}")
