"""GPU parity of the sm_100a tile kernels against the reference's own
outputs (golden fixtures from the unmodified reference) and against a torch
fp32 restatement at larger sizes.  Tolerances: rel-Fro
<= 1e-2 on O/dQ/dK/dV, LSE max-abs <= 1e-3 — bf16 inputs and P, fp32
accumulation vs the fp64 reference."""

from pathlib import Path

import numpy as np
import pytest
import torch

from gpu_util import bf16_from_bits, max_abs, ref_attention, rel_fro, uniform

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
REL_TOL = 1e-2
LSE_TOL = 1e-3


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_15758_b200 import ops as _ops
    return _ops


@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("n", [64, 128])
def test_umma_descriptor_selftest(ops, b_mn, n):
    a = uniform((128, 128), 1)
    b = uniform((128, n) if b_mn else (n, 128), 2)
    d = ops.selftest_umma(a, b, b_mn)
    want = a.float() @ (b.float() if b_mn else b.float().T)
    torch.cuda.synchronize()
    assert max_abs(d, want) < 1e-3, max_abs(d, want)


GOLD_CASES = ["n256_h64_causal", "n256_h64_none_s1", "n128_h128_causal", "n320_h128_none"]


@pytest.mark.parametrize("tag", GOLD_CASES)
def test_forward_matches_reference_golden(ops, tag):
    g = np.load(GOLD / "gpu_parity.npz")
    n, h, causal, scale = g[f"{tag}_meta"]
    q, k, v = (bf16_from_bits(g[f"{tag}_{x}"]).cuda()[None] for x in "qkv")
    o, lse = ops.tile_forward(q, k, v, causal=bool(causal), scale=float(scale))
    want_o = torch.from_numpy(g[f"{tag}_o"]).cuda()
    want_lse = torch.from_numpy(g[f"{tag}_lse"]).cuda()
    assert rel_fro(o[0], want_o) < REL_TOL
    assert max_abs(lse[0], want_lse) < LSE_TOL
    ob, lse2 = ops.tile_forward(q, k, v, causal=bool(causal), scale=float(scale),
                                out_dtype=torch.bfloat16)
    assert rel_fro(ob[0].float(), want_o) < REL_TOL
    assert torch.equal(lse, lse2)


@pytest.mark.parametrize("h", [64, 96, 128])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("nq,nk", [(128, 128), (200, 200), (1024, 1024), (384, 1000), (7, 9)])
def test_forward_vs_torch(ops, h, causal, nq, nk):
    bh = 3
    q, k, v = uniform((bh, nq, h), 10), uniform((bh, nk, h), 11), uniform((bh, nk, h), 12)
    scale = h ** -0.5
    # causal with nq != nk: queries are the LAST nq positions of the key range
    qi = ops.TokenIndex.contiguous(nq, start=max(nk - nq, 0))
    o, lse = ops.tile_forward(q, k, v, causal=causal, scale=scale, q_index=qi)
    q_idx = torch.arange(nq) + max(nk - nq, 0)
    want_o, want_lse = ref_attention(q, k, v, causal, scale, q_idx=q_idx)
    torch.cuda.synchronize()
    assert rel_fro(o, want_o) < REL_TOL
    fin = torch.isfinite(want_lse)
    assert torch.equal(fin, torch.isfinite(lse))
    assert max_abs(lse[fin], want_lse[fin]) < LSE_TOL


def test_forward_unit_scale_peaky(ops):
    """Reference default scale = 1.0 (common.py:26): large scores."""
    q, k, v = uniform((2, 512, 128), 20), uniform((2, 512, 128), 21), uniform((2, 512, 128), 22)
    o, lse = ops.tile_forward(q, k, v, causal=True, scale=1.0)
    want_o, want_lse = ref_attention(q, k, v, True, 1.0)
    assert rel_fro(o, want_o) < REL_TOL
    assert max_abs(lse, want_lse) < LSE_TOL


def test_forward_index_subsets_array_mode(ops):
    """Global indices drive masking, not local positions
    (reference test_attention.py:136-145), incl. fully masked rows."""
    rng = np.random.default_rng(5)
    q_idx = np.sort(rng.choice(600, size=150, replace=False))
    k_idx = np.sort(rng.choice(np.arange(20, 600), size=260, replace=False))
    qi = ops.TokenIndex.from_indices(q_idx)
    ki = ops.TokenIndex.from_indices(k_idx)
    assert qi.is_array and ki.is_array
    q, k, v = uniform((2, 150, 64), 30), uniform((2, 260, 64), 31), uniform((2, 260, 64), 32)
    o, lse = ops.tile_forward(q, k, v, causal=True, scale=0.125, q_index=qi, k_index=ki)
    want_o, want_lse = ref_attention(q, k, v, True, 0.125, torch.from_numpy(q_idx),
                                     torch.from_numpy(k_idx))
    empty = q_idx < k_idx[0]
    assert empty.any()
    assert torch.all(torch.isneginf(lse[:, torch.from_numpy(empty)]))
    assert torch.all(o[:, torch.from_numpy(empty)] == 0)
    live = torch.from_numpy(~empty)
    assert rel_fro(o[:, live], want_o[:, live]) < REL_TOL
    assert max_abs(lse[:, live], want_lse[:, live]) < LSE_TOL


@pytest.mark.parametrize("pr,pc", [(2, 2), (2, 4), (4, 2)])
def test_forward_blocked_cyclic_maps(ops, pr, pc):
    """The 2D gathered orders: query block c' holds tokens r + Pr c' + P i,
    key block r' holds c + Pc r' + P i."""
    P, L, h = pr * pc, 256, 128
    N = P * L
    r, c = pr - 1, 0
    qi = ops.TokenIndex.blocked([r + pr * cc for cc in range(pc)], P, L)
    ki = ops.TokenIndex.blocked([c + pc * rr for rr in range(pr)], P, L)
    q, k, v = uniform((2, pc * L, h), 40), uniform((2, pr * L, h), 41), uniform((2, pr * L, h), 42)
    o, lse = ops.tile_forward(q, k, v, causal=True, scale=h ** -0.5, q_index=qi, k_index=ki)
    want_o, want_lse = ref_attention(q, k, v, True, h ** -0.5, torch.from_numpy(qi.host()),
                                     torch.from_numpy(ki.host()))
    fin = torch.isfinite(want_lse)
    assert torch.equal(fin, torch.isfinite(lse))
    assert rel_fro(o[fin], want_o[fin]) < REL_TOL
    assert max_abs(lse[fin], want_lse[fin]) < LSE_TOL
    # the same maps through the array path agree up to bf16 rounding of P:
    # the array path evaluates every exponential on MUFU and visits the key
    # tiles in another order (another stale running max), the affine path
    # offloads a quarter of the exponentials to the cubic exp2
    o2, lse2 = ops.tile_forward(q, k, v, causal=True, scale=h ** -0.5, q_index=qi.as_array("cuda"),
                                k_index=ki.as_array("cuda"))
    assert max_abs(o2, o) < 5e-3 and max_abs(lse2[fin], lse[fin]) < 5e-4


def test_forward_continuation(ops):
    """Two calls over split key ranges equal one call
    (reference test_kernels.py:124-137)."""
    q, k, v = uniform((2, 300, 128), 50), uniform((2, 700, 128), 51), uniform((2, 700, 128), 52)
    qi = ops.TokenIndex.contiguous(300, start=400)
    whole_o, whole_lse = ops.tile_forward(q, k, v, causal=True, scale=0.1, q_index=qi)
    o, lse = ops.tile_forward(q, k[:, :256], v[:, :256], causal=True, scale=0.1, q_index=qi,
                              k_index=ops.TokenIndex.contiguous(256))
    ops.tile_forward(q, k[:, 256:], v[:, 256:], causal=True, scale=0.1, q_index=qi,
                     k_index=ops.TokenIndex.contiguous(444, start=256), out=o, lse=lse,
                     accumulate=True)
    assert max_abs(o, whole_o) < 1e-3
    assert max_abs(lse, whole_lse) < 1e-3


@pytest.mark.parametrize("kparts", [1, 2, 3, 4, 5, 8, 16])
def test_lse_merge_matches_oracle(ops, kparts):
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle import attn2d_oracle as orc
    rows, h = 333, 128
    g = torch.Generator().manual_seed(kparts)
    o_parts = torch.randn((kparts, rows, h), generator=g)
    lse_parts = torch.randn((kparts, rows), generator=g) * 3
    lse_parts[0, :5] = float("-inf")
    if kparts > 1:
        lse_parts[:, 7] = float("-inf")
    o, lse = ops.lse_merge(o_parts.cuda(), lse_parts.cuda(), out_dtype=torch.float32)
    want_o, want_lse = orc.lse_merge(list(o_parts.double().numpy()),
                                     list(lse_parts.double().numpy()))
    assert np.abs(o.cpu().numpy() - want_o).max() < 1e-5
    fin = np.isfinite(want_lse)
    assert np.array_equal(fin, np.isfinite(lse.cpu().numpy()))
    assert np.abs(lse.cpu().numpy()[fin] - want_lse[fin]).max() < 1e-5


# --------------------------------------------------------------------------
# backward
# --------------------------------------------------------------------------

def _run_backward(ops, q, k, v, dout, causal, scale, q_index=None, k_index=None):
    o, lse = ops.tile_forward(q, k, v, causal=causal, scale=scale, q_index=q_index,
                              k_index=k_index, out_dtype=torch.bfloat16)
    delta = ops.bwd_preprocess(o, dout)
    dq_acc, dk, dv = ops.tile_backward(q, k, v, dout, lse, delta, causal=causal, scale=scale,
                                       q_index=q_index, k_index=k_index)
    dq = ops.bwd_finalize(dq_acc, scale, dtype=torch.float32)
    return o, lse, dq, dk, dv


@pytest.mark.parametrize("tag", GOLD_CASES)
def test_backward_matches_reference_golden(ops, tag):
    g = np.load(GOLD / "gpu_parity.npz")
    n, h, causal, scale = g[f"{tag}_meta"]
    q, k, v, dout = (bf16_from_bits(g[f"{tag}_{x}"]).cuda()[None] for x in ("q", "k", "v", "dout"))
    _, _, dq, dk, dv = _run_backward(ops, q, k, v, dout, bool(causal), float(scale))
    for name, got in (("dq", dq), ("dk", dk), ("dv", dv)):
        want = torch.from_numpy(g[f"{tag}_{name}"]).cuda()
        assert rel_fro(got[0], want) < REL_TOL, (name, rel_fro(got[0], want))


@pytest.mark.parametrize("h", [32, 64, 96, 128])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("n", [128, 200, 1024])
def test_backward_vs_torch(ops, h, causal, n):
    from gpu_util import ref_attention_grad
    bh = 3
    q, k, v, dout = (uniform((bh, n, h), 60 + i) for i in range(4))
    scale = h ** -0.5
    _, _, dq, dk, dv = _run_backward(ops, q, k, v, dout, causal, scale)
    wq, wk, wv = ref_attention_grad(q, k, v, dout, causal, scale)
    torch.cuda.synchronize()
    for name, got, want in (("dq", dq, wq), ("dk", dk, wk), ("dv", dv, wv)):
        assert rel_fro(got, want) < REL_TOL, (name, rel_fro(got, want))


def test_backward_key_subsets_are_partial_sums(ops):
    """Key-subset calls with global statistics sum to the full gradient
    (reference test_attention.py:305-328)."""
    n, h = 512, 128
    q, k, v, dout = (uniform((2, n, h), 70 + i) for i in range(4))
    scale = h ** -0.5
    o, lse, dq, dk, dv = _run_backward(ops, q, k, v, dout, True, scale)
    delta = ops.bwd_preprocess(o, dout)
    dq_acc = torch.zeros((2, n, h), device="cuda")
    dks, dvs = [], []
    for lo, hi in ((0, 256), (256, 512)):
        _, dk_p, dv_p = ops.tile_backward(q, k[:, lo:hi], v[:, lo:hi], dout, lse, delta,
                                          causal=True, scale=scale, dq_acc=dq_acc,
                                          k_index=ops.TokenIndex.contiguous(hi - lo, start=lo))
        dks.append(dk_p)
        dvs.append(dv_p)
    dq2 = ops.bwd_finalize(dq_acc, scale, dtype=torch.float32)
    assert max_abs(dq2, dq) < 1e-4
    assert max_abs(torch.cat(dks, 1), dk) < 1e-4
    assert max_abs(torch.cat(dvs, 1), dv) < 1e-4


@pytest.mark.parametrize("pr,pc", [(2, 2), (2, 4)])
def test_backward_blocked_cyclic_maps(ops, pr, pc):
    from gpu_util import ref_attention
    P, L, h = pr * pc, 256, 128
    r, c = 1, pc - 1
    qi = ops.TokenIndex.blocked([r + pr * cc for cc in range(pc)], P, L)
    ki = ops.TokenIndex.blocked([c + pc * rr for rr in range(pr)], P, L)
    q, k, v = uniform((1, pc * L, h), 80), uniform((1, pr * L, h), 81), uniform((1, pr * L, h), 82)
    dout = uniform((1, pc * L, h), 83)
    scale = h ** -0.5
    qi_t, ki_t = torch.from_numpy(qi.host()), torch.from_numpy(ki.host())
    # global statistics of these query rows against THESE keys only (a tile of
    # the grid), then the gradient of that partial attention
    qf = q.float().requires_grad_(True)
    kf = k.float().requires_grad_(True)
    vf = v.float().requires_grad_(True)
    o_ref, lse_ref = ref_attention(qf, kf, vf, True, scale, qi_t, ki_t)
    live = torch.isfinite(lse_ref)
    (o_ref * dout.float() * live[..., None]).sum().backward()
    _, _, dq, dk, dv = _run_backward(ops, q, k, v, dout * live[..., None], True, scale, qi, ki)
    assert rel_fro(dq[live], qf.grad[live]) < REL_TOL
    assert rel_fro(dk, kf.grad) < REL_TOL
    assert rel_fro(dv, vf.grad) < REL_TOL


@pytest.mark.parametrize("b_mn", [False, True])
def test_umma_a_operand_from_tmem(ops, b_mn):
    """tcgen05.mma with A in TMEM (bf16 pairs per 32-bit column)."""
    a = uniform((128, 128), 3)
    b = uniform((128, 128), 4)
    d = ops.selftest_umma(a, b, 2 | int(b_mn))
    want = a.float() @ (b.float() if b_mn else b.float().T)
    torch.cuda.synchronize()
    assert max_abs(d, want) < 1e-3, max_abs(d, want)


@pytest.mark.parametrize("h", [64, 128])
@pytest.mark.parametrize("array_mode", [False, True])
def test_no_uninitialised_reads_and_deterministic(ops, h, array_mode):
    """Outputs pre-filled with NaN and SMEM/TMEM of every SM poisoned with NaN
    before each launch: every output element must be written, and the result
    must be bitwise identical across runs (no read of on-chip memory the
    kernel did not write; no phase-parity race on the mbarriers)."""
    rng = np.random.default_rng(11)
    nq, nk = 300, 420
    if array_mode:
        q_idx = np.sort(rng.choice(1000, size=nq, replace=False))
        k_idx = np.sort(rng.choice(np.arange(30, 1000), size=nk, replace=False))
        qi, ki = ops.TokenIndex.from_indices(q_idx), ops.TokenIndex.from_indices(k_idx)
    else:
        qi, ki = ops.TokenIndex.contiguous(nq, 500), ops.TokenIndex.contiguous(nk, 100)
    q, dout = uniform((2, nq, h), 70), uniform((2, nq, h), 71)
    k, v = uniform((2, nk, h), 72), uniform((2, nk, h), 73)
    runs = []
    for poison in (0, 3, 3):
        o = torch.full((2, nq, h), float("nan"), device="cuda")
        lse = torch.full((2, nq), float("nan"), device="cuda")
        ops.debug_poison(poison)
        ops.tile_forward(q, k, v, causal=True, scale=0.1, q_index=qi, k_index=ki, out=o, lse=lse)
        delta = ops.bwd_preprocess(o.to(torch.bfloat16), dout)
        dq_acc = torch.zeros((2, nq, h), device="cuda")
        dk = torch.full((2, nk, h), float("nan"), device="cuda")
        dv = torch.full((2, nk, h), float("nan"), device="cuda")
        ops.debug_poison(poison)
        ops.tile_backward(q, k, v, dout, lse, delta, causal=True, scale=0.1, q_index=qi,
                          k_index=ki, dq_acc=dq_acc, dk=dk, dv=dv)
        torch.cuda.synchronize()
        for name, t in (("o", o), ("dq", dq_acc), ("dk", dk), ("dv", dv)):
            assert not torch.isnan(t).any(), name
        assert not torch.isnan(lse).any()
        runs.append((o, lse, dq_acc, dk, dv))
    # o, lse, dk, dv are bitwise reproducible; dq_acc is summed by TMA
    # reduce-adds from many CTAs in hardware order (fp32 non-associativity)
    for run in runs[1:]:
        for i, (a, b) in enumerate(zip(runs[0], run)):
            if i == 2:
                assert rel_fro(a, b) < 1e-5
            else:
                assert torch.equal(a, b)


@pytest.mark.parametrize("m,m_kv", [(8, 2), (4, 1)])
@pytest.mark.parametrize("causal", [False, True])
def test_grouped_query_attention_fwd_bwd(ops, m, m_kv, causal):
    """GQA / MQA: query head j reads k/v head j // (m / m_kv)
    inside the kernels (kv_group); dK / dV are summed over each group."""
    from paper_2503_15758_b200 import functional
    from gpu_util import ref_attention_grad
    b, n, h = 2, 384, 128
    q, do = uniform((b, m, n, h), 71), uniform((b, m, n, h), 72)
    k, v = uniform((b, m_kv, n, h), 73), uniform((b, m_kv, n, h), 74)
    scale = h ** -0.5
    qg, kg, vg = (x.clone().requires_grad_(True) for x in (q, k, v))
    o = functional.attention(qg, kg, vg, causal=causal, scale=scale)
    o.backward(do)
    g = m // m_kv
    rep = lambda x: x.repeat_interleave(g, dim=1).reshape(b * m, n, h)  # noqa: E731
    want_o, _ = ref_attention(q.reshape(b * m, n, h), rep(k), rep(v), causal, scale)
    assert rel_fro(o.reshape(b * m, n, h), want_o) < REL_TOL
    wq, wk, wv = ref_attention_grad(q.reshape(b * m, n, h), rep(k), rep(v),
                                    do.reshape(b * m, n, h), causal, scale)
    wk = wk.reshape(b, m_kv, g, n, h).sum(2)
    wv = wv.reshape(b, m_kv, g, n, h).sum(2)
    assert rel_fro(qg.grad.reshape(b * m, n, h), wq) < REL_TOL
    assert rel_fro(kg.grad, wk) < REL_TOL
    assert rel_fro(vg.grad, wv) < REL_TOL


@pytest.mark.parametrize("h", [4, 32, 48, 80, 96, 104])
def test_other_head_dims(ops, h):
    """Head dims other than 64 / 128, incl. the reference's H=80 / 96 presets
    (costmodel.py:73-79) natively (TMA zero fill inside the 64 / 128-wide
    tiles) and h=4 (the reference tests' size) padded to 8."""
    from paper_2503_15758_b200 import functional
    from gpu_util import ref_attention_grad
    bh, n = 3, 256
    q, k, v, do = (uniform((bh, n, h), 80 + i) for i in range(4))
    scale = h ** -0.5
    qg, kg, vg = (x.clone().requires_grad_(True) for x in (q, k, v))
    o = functional.attention(qg, kg, vg, causal=True, scale=scale)
    o.backward(do)
    want_o, _ = ref_attention(q, k, v, True, scale)
    assert o.shape == q.shape and rel_fro(o, want_o) < REL_TOL
    wq, wk, wv = ref_attention_grad(q, k, v, do, True, scale)
    for got, want in ((qg.grad, wq), (kg.grad, wk), (vg.grad, wv)):
        assert rel_fro(got, want) < REL_TOL


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("h", [64, 128])
@pytest.mark.parametrize("causal", [False, True])
def test_forward_growing_scores_move_the_running_max(ops, causal, h, dt):
    """Scores that grow by ~2^100 along the key sweep: the forward's running
    max (taken from the first visible tile, moved only when a tile's sum
    nears overflow: 2^64 with bf16 P, 2^15 with fp16 P) must re-base exactly;
    compared with the fp32 reference."""
    bh, n = 2, 1024
    g = torch.Generator(device="cpu").manual_seed(7)
    u = torch.randn((h,), generator=g)
    u = u / u.norm()
    a = torch.linspace(0.5, 1.0, n)[:, None]                  # query rows
    b = torch.linspace(-10.0, 90.0, n)[:, None]               # key rows: growing scores
    noise = lambda: 0.05 * torch.randn((n, h), generator=g)   # noqa: E731
    q = (a * u + noise()).expand(bh, n, h).contiguous().to("cuda", dt)
    k = (b * u + noise()).expand(bh, n, h).contiguous().to("cuda", dt)
    v = uniform((bh, n, h), 91).to(dt)
    o, lse = ops.tile_forward(q, k, v, causal=causal, scale=1.0, out_dtype=torch.float32)
    want_o, want_lse = ref_attention(q, k, v, causal, 1.0)
    assert torch.isfinite(o).all() and torch.isfinite(lse).all()
    assert rel_fro(o, want_o) < REL_TOL
    assert max_abs(lse, want_lse) < 1e-3 * max(1.0, float(want_lse.abs().max()))


@pytest.mark.parametrize("n,bh", [(32768, 2), (131072, 1)])
def test_full_size_row_and_key_sampled_parity(ops, n, bh):
    """C2 (N=32768) and the metric size (N=131072), H=128, causal, with fewer
    heads, against an fp64 reference evaluated chunk-wise on the GPU (SURVEY
    §8c "large N" protocol): LSE of every row, O / dQ on sampled query rows,
    dK / dV on sampled key rows."""
    from paper_2503_15758_b200 import functional
    h = 128
    scale = h ** -0.5
    q, k, v, do = (uniform((bh, n, h), 120 + i) for i in range(4))
    qg, kg, vg = (x.clone().requires_grad_(True) for x in (q, k, v))
    o = functional.attention(qg, kg, vg, causal=True, scale=scale)
    o.backward(do)
    _, lse = ops.tile_forward(q, k, v, causal=True, scale=scale, out_dtype=torch.bfloat16)
    qd, kd, vd, dod = (x.double() for x in (q, k, v, do))
    kidx = torch.arange(n, device="cuda")
    lse_ref = torch.empty((bh, n), dtype=torch.float64, device="cuda")
    o_ref = torch.empty((bh, n, h), dtype=torch.float64, device="cuda")
    for r0 in range(0, n, 2048):
        s = torch.einsum("bqh,bkh->bqk", qd[:, r0:r0 + 2048], kd) * scale  # [bh, 2048, n]
        s = s.masked_fill(kidx[None, None, :] > (r0 + torch.arange(2048, device="cuda"))[None, :, None],
                          float("-inf"))
        lse_ref[:, r0:r0 + 2048] = torch.logsumexp(s, -1)
        o_ref[:, r0:r0 + 2048] = torch.einsum("bqk,bkh->bqh",
                                              torch.exp(s - lse_ref[:, r0:r0 + 2048, None]), vd)
    assert max_abs(lse, lse_ref) < LSE_TOL
    delta_ref = (o_ref * dod).sum(-1)
    g = torch.Generator(device="cpu").manual_seed(5)
    rows = torch.randint(0, n, (96,), generator=g).cuda()
    keys = torch.randint(0, n, (96,), generator=g).cuda()
    # sampled query rows: O and dQ
    s = torch.einsum("bqh,bkh->bqk", qd[:, rows], kd) * scale
    s = s.masked_fill(kidx[None, None, :] > rows[None, :, None], float("-inf"))
    p = torch.exp(s - lse_ref[:, rows, None])
    dp = torch.einsum("bqh,bkh->bqk", dod[:, rows], vd)
    dq_ref = torch.einsum("bqk,bkh->bqh", p * (dp - delta_ref[:, rows, None]), kd) * scale
    assert rel_fro(o[:, rows], o_ref[:, rows]) < REL_TOL
    assert rel_fro(qg.grad[:, rows], dq_ref) < REL_TOL
    # sampled key rows: dK and dV over every query
    s = torch.einsum("bqh,bkh->bqk", qd, kd[:, keys]) * scale
    s = s.masked_fill(keys[None, None, :] > kidx[None, :, None], float("-inf"))
    p = torch.exp(s - lse_ref[:, :, None])
    dp = torch.einsum("bqh,bkh->bqk", dod, vd[:, keys])
    dk_ref = torch.einsum("bqk,bqh->bkh", p * (dp - delta_ref[:, :, None]), qd) * scale
    dv_ref = torch.einsum("bqk,bqh->bkh", p, dod)
    assert rel_fro(kg.grad[:, keys], dk_ref) < REL_TOL
    assert rel_fro(vg.grad[:, keys], dv_ref) < REL_TOL


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("h", [64, 128])
@pytest.mark.parametrize("col", [270, 271, 300, 330, 383])
def test_forward_single_huge_score_on_any_column(ops, col, h, dt):
    """One key whose score exceeds every earlier tile's by ~2^200, placed on
    a column the forward evaluates with the FMA-pipe polynomial (270, 271)
    or with MUFU (300, 330, 383), in either key half of its tile: the
    overflow guard must catch it either way."""
    bh, n = 1, 512
    g = torch.Generator(device="cpu").manual_seed(11)
    u = torch.randn((h,), generator=g)
    u = u / u.norm()
    q = (u + 0.01 * torch.randn((n, h), generator=g))[None].contiguous()
    k = (0.01 * torch.randn((n, h), generator=g))[None].contiguous()
    k[0, col] = 140.0 * u
    q, k = q.to("cuda", dt), k.to("cuda", dt)
    v = uniform((bh, n, h), 93).to(dt)
    for causal in (False, True):
        o, lse = ops.tile_forward(q, k, v, causal=causal, scale=1.0, out_dtype=torch.float32)
        want_o, want_lse = ref_attention(q, k, v, causal, 1.0)
        assert torch.isfinite(o).all() and torch.isfinite(lse).all()
        assert rel_fro(o, want_o) < REL_TOL, (causal, rel_fro(o, want_o))
        assert max_abs(lse, want_lse) < 1e-3 * max(1.0, float(want_lse.abs().max()))


@pytest.mark.parametrize("causal", [False, True])
def test_backward_accumulate_mode_adds_to_existing_dkv(ops, causal):
    """accumulate_dkv (ABI v3): two key-disjoint query subsets accumulated
    into one fp32 dK/dV buffer equal the full-query backward (the ring's and
    attn2d_o's hop accumulation, reference ring.py:118-143)."""
    bh, n, h = 2, 384, 128
    scale = h ** -0.5
    q, k, v, do = (uniform((bh, n, h), s) for s in (51, 52, 53, 54))
    o, lse = ops.tile_forward(q, k, v, causal=causal, scale=scale, out_dtype=torch.bfloat16)
    delta = ops.bwd_preprocess(o, do)
    _, dk_full, dv_full = ops.tile_backward(q, k, v, do, lse, delta, causal=causal, scale=scale)
    dk = torch.full((bh, n, h), 0.25, device="cuda")
    dv = torch.full((bh, n, h), -0.5, device="cuda")
    dk0, dv0 = dk.clone(), dv.clone()
    for a, b in ((0, 128), (128, 384)):   # query row subsets (global positions a..b-1)
        qi = ops.TokenIndex.contiguous(b - a, a)
        dq_part = torch.zeros((bh, b - a, h), device="cuda")
        ops.tile_backward(q[:, a:b].contiguous(), k, v, do[:, a:b].contiguous(),
                          lse[:, a:b].contiguous(), delta[:, a:b].contiguous(), causal=causal,
                          scale=scale, q_index=qi, dq_acc=dq_part, dk=dk, dv=dv,
                          accumulate_dkv=True)
    torch.cuda.synchronize()
    assert rel_fro(dk - dk0, dk_full) < 1e-5
    assert rel_fro(dv - dv0, dv_full) < 1e-5


def test_backward_without_query_rows_writes_zero_dkv(ops):
    """nq == 0: nothing attends these keys, dK / dV are zero (reference
    attention.py:250-252), in both output dtypes."""
    bh, nk, h = 2, 200, 64
    k, v = uniform((bh, nk, h), 61), uniform((bh, nk, h), 62)
    q = torch.empty((bh, 0, h), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((bh, 0), device="cuda")
    for dt in (torch.float32, torch.bfloat16):
        dk = torch.full((bh, nk, h), 7.0, dtype=dt, device="cuda")
        dv = torch.full((bh, nk, h), 7.0, dtype=dt, device="cuda")
        ops.tile_backward(q, k, v, q, lse, lse, causal=True, scale=0.125, dk=dk, dv=dv)
        torch.cuda.synchronize()
        assert bool((dk == 0).all()) and bool((dv == 0).all())


def test_forward_without_heads_or_rows_is_a_no_op(ops):
    """bh == 0 and nq == 0 launch nothing and succeed (a2d_tile_fwd)."""
    for bh, nq in ((0, 128), (2, 0)):
        q = torch.empty((bh, nq, 64), dtype=torch.bfloat16, device="cuda")
        k = uniform((bh, 64, 64), 63) if bh else torch.empty((0, 64, 64), dtype=torch.bfloat16,
                                                              device="cuda")
        o, lse = ops.tile_forward(q, k, k, causal=True, scale=0.125)
        assert o.shape == (bh, nq, 64) and lse.shape == (bh, nq)


@pytest.mark.parametrize("m,m_kv", [(4, 4), (4, 2)])
@pytest.mark.parametrize("causal", [False, True])
def test_fp16_attention_fwd_bwd(ops, causal, m, m_kv):
    """fp16 operands end to end (in_dtype A2D_F16: fp16 TMA maps, kind::f16
    MMAs with fp16 A/B, fp16 P and dS): functional.attention forward and
    backward in fp16 against the fp32 reference, GQA included."""
    from paper_2503_15758_b200 import functional
    from gpu_util import ref_attention_grad
    n, h = 640, 128
    scale = h ** -0.5
    q, do = (uniform((m, n, h), 210 + i).to(torch.float16) for i in range(2))
    k, v = (uniform((m_kv, n, h), 220 + i).to(torch.float16) for i in range(2))
    qg, kg, vg = (x.clone().requires_grad_(True) for x in (q, k, v))
    o = functional.attention(qg, kg, vg, causal=causal, scale=scale)
    o.backward(do)
    assert o.dtype == torch.float16 and qg.grad.dtype == torch.float16
    rep = m // m_kv
    kr, vr = k.repeat_interleave(rep, 0), v.repeat_interleave(rep, 0)
    want_o, _ = ref_attention(q, kr, vr, causal, scale)
    dq, dk, dv = ref_attention_grad(q, kr, vr, do, causal, scale)
    dk = dk.view(m_kv, rep, n, h).sum(1)
    dv = dv.view(m_kv, rep, n, h).sum(1)
    assert rel_fro(o, want_o) < REL_TOL
    for got, want in ((qg.grad, dq), (kg.grad, dk), (vg.grad, dv)):
        assert rel_fro(got, want) < REL_TOL, rel_fro(got, want)


def test_fp16_merge_and_finalize_outputs(ops):
    """lse_merge and bwd_finalize write fp16 as they write bf16 (A2D_F16)."""
    rows, h = 300, 128
    o_parts = torch.randn((3, rows, h), device="cuda")
    lse_parts = torch.randn((3, rows), device="cuda")
    o16, lse16 = ops.lse_merge(o_parts, lse_parts, out_dtype=torch.float16)
    o32, lse32 = ops.lse_merge(o_parts, lse_parts, out_dtype=torch.float32)
    assert o16.dtype == torch.float16 and torch.equal(lse16, lse32)
    assert max_abs(o16.float(), o32) <= float(o32.abs().max()) * 2 ** -10
    acc = torch.randn((2, rows, h), device="cuda")
    dq = ops.bwd_finalize(acc, 0.5, dtype=torch.float16)
    assert torch.equal(dq, (acc * 0.5).to(torch.float16))
