"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Outputs `tests/golden/*.npz`.  Everything is produced through the reference's
public API (attn2d.kernels / attn2d.attention / attn2d.strategies), numpy
kernel backend, float64.  Inputs follow the reference convention
`np.random.default_rng(seed).uniform(-1, 1, (n, h))` in q, k, v, d_out order
(cli.py:56-61, test_strategies.py:16-22).  For the GPU parity fixtures the
inputs are rounded once to bf16 and the same rounded values are fed to the
reference (SURVEY.md §8c parity protocol); they are stored as raw bf16 bits.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ["ATTN2D_KERNEL"] = "numpy"
sys.path.insert(0, str(REF))

from attn2d import kernels  # noqa: E402
from attn2d.attention import (MaskKind, MaskSpec, PartialAttn, TokenShard,  # noqa: E402
                              attn_fix, count_unmasked, finalize,
                              flash_attn_backward, flash_attn_forward,
                              reference_attention)
from attn2d.strategies import DistAttnConfig, run_backward, run_forward  # noqa: E402

kernels.use_backend("numpy")


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float64 values."""
    u = a.astype(np.float32).view(np.uint32)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.view(np.float32).astype(np.float64)


def bf16_bits(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)


def gen(n, h, seed, nk=None):
    rng = np.random.default_rng(seed)
    nk = n if nk is None else nk
    q = rng.uniform(-1.0, 1.0, (n, h))
    k = rng.uniform(-1.0, 1.0, (nk, h))
    v = rng.uniform(-1.0, 1.0, (nk, h))
    d_out = rng.uniform(-1.0, 1.0, (n, h))
    return q, k, v, d_out


def random_problem(seed, nq=7, nk=9, h=5):
    """test_kernels.py:17-27: random rows with sorted index subsets."""
    rng = np.random.default_rng(seed)
    q = rng.uniform(-1, 1, (nq, h))
    k = rng.uniform(-1, 1, (nk, h))
    v = rng.uniform(-1, 1, (nk, h))
    q_idx = np.sort(rng.choice(32, size=nq, replace=False)).astype(np.int64)
    rest = np.sort(rng.choice(np.arange(1, 32), size=nk - 1, replace=False))
    k_idx = np.concatenate([[0], rest]).astype(np.int64)
    return q, k, v, q_idx, k_idx


def tile_cases():
    out = {}
    for causal in (False, True):
        q, k, v, qi, ki = random_problem(11)
        m = np.full(q.shape[0], -np.inf)
        nacc = np.zeros_like(q)
        d = np.zeros(q.shape[0])
        kernels.flash_forward(q, k, v, qi, ki, causal, 1.0, 64, m, nacc, d)
        live = d > 0
        o = np.zeros_like(q)
        o[live] = nacc[live] / d[live, None]
        d_out = np.random.default_rng(13).uniform(-1, 1, q.shape)
        dq, dk, dv = (np.zeros_like(q), np.zeros_like(k), np.zeros_like(v))
        kernels.flash_backward(q, k, v, o, d_out, m, d, qi, ki, causal, 1.0, dq, dk, dv)
        tag = "causal" if causal else "none"
        out.update({f"{tag}_q": q, f"{tag}_k": k, f"{tag}_v": v, f"{tag}_q_idx": qi,
                    f"{tag}_k_idx": ki, f"{tag}_m": m, f"{tag}_n": nacc, f"{tag}_d": d,
                    f"{tag}_o": o, f"{tag}_dout": d_out, f"{tag}_dq": dq, f"{tag}_dk": dk,
                    f"{tag}_dv": dv})
    # SPEC.md:132-133 known answer: q=[0], k=[0,1], v=[[2],[4]], zero q/k
    part = flash_attn_forward(TokenShard(np.zeros((1, 1)), [0]),
                              TokenShard(np.zeros((2, 1)), [0, 1]),
                              TokenShard(np.array([[2.0], [4.0]]), [0, 1]),
                              MaskSpec.none(), 1.0, 1)
    out.update(kat_tile_m=part.m, kat_tile_n=part.n, kat_tile_d=part.d)
    # masked-row case (test_attention.py:147-157)
    rng = np.random.default_rng(46)
    q = rng.uniform(-1, 1, (2, 2))
    k = np.random.default_rng(47).uniform(-1, 1, (2, 2))
    v = np.random.default_rng(48).uniform(-1, 1, (2, 2))
    part = flash_attn_forward(TokenShard(q, [0, 8]), TokenShard(k, [4, 5]),
                              TokenShard(v, [4, 5]), MaskSpec.causal())
    out.update(masked_q=q, masked_k=k, masked_v=v, masked_m=part.m,
               masked_n=part.n, masked_d=part.d)
    # index subsets (test_attention.py:136-145)
    qi, ki = np.array([3, 9, 17]), np.array([2, 9, 12, 20])
    q = np.random.default_rng(43).uniform(-1, 1, (3, 3))
    k = np.random.default_rng(44).uniform(-1, 1, (4, 3))
    v = np.random.default_rng(45).uniform(-1, 1, (4, 3))
    part = flash_attn_forward(TokenShard(q, qi), TokenShard(k, ki), TokenShard(v, ki),
                              MaskSpec.causal())
    out.update(subset_q=q, subset_k=k, subset_v=v, subset_q_idx=qi, subset_k_idx=ki,
               subset_o=finalize(part), subset_lse=part.logsumexp)
    np.savez_compressed(OUT / "tile_small.npz", **out)


def merge_cases():
    out = {}
    # (0,[[1]],1) (+) (0,[[3]],1) -> (0,[[4]],2)
    a = PartialAttn(np.array([0.0]), np.array([[1.0]]), np.array([1.0]))
    b = PartialAttn(np.array([0.0]), np.array([[3.0]]), np.array([1.0]))
    r = attn_fix(a, b)
    out.update(kat_m=r.m, kat_n=r.n, kat_d=r.d)
    # random 4-way partials over disjoint key subsets, merged left to right
    q, k, v, _ = gen(6, 3, seed=60, nk=16)
    cuts = [0, 3, 7, 12, 16]
    parts = []
    for i in range(4):
        idx = np.arange(cuts[i], cuts[i + 1])
        parts.append(flash_attn_forward(TokenShard(q, np.arange(6) + 8),
                                        TokenShard(k[idx], idx), TokenShard(v[idx], idx),
                                        MaskSpec.causal()))
    acc = parts[0]
    for p in parts[1:]:
        acc = attn_fix(acc, p)
    for i, p in enumerate(parts):
        out[f"part{i}_m"], out[f"part{i}_n"], out[f"part{i}_d"] = p.m, p.n, p.d
    out.update(fold_m=acc.m, fold_n=acc.n, fold_d=acc.d, fold_o=finalize(acc),
               fold_lse=acc.logsumexp)
    np.savez_compressed(OUT / "merge_small.npz", **out)


def strategy_cases():
    out = {}
    for name in ("attn2d_no", "attn2d_o", "ring"):
        for causal in (False, True):
            n, h, p = 32, 4, 4
            mask = MaskKind.CAUSAL if causal else MaskKind.NONE
            cfg = DistAttnConfig(n=n, h=h, p=p, mask=mask)
            q, k, v, d_out = gen(n, h, seed=n * 31 + p)
            fwd = run_forward(name, cfg, q, k, v)
            bwd = run_backward(name, cfg, fwd.saved, d_out)
            tag = f"{name}_{'causal' if causal else 'none'}"
            out.update({f"{tag}_o": fwd.o, f"{tag}_dq": bwd.dq, f"{tag}_dk": bwd.dk,
                        f"{tag}_dv": bwd.dv,
                        f"{tag}_scores": np.array([fwd.score_elements[c] for c in
                                                   sorted(fwd.score_elements)])})
    q, k, v, d_out = gen(32, 4, seed=32 * 31 + 4)
    out.update(q=q, k=k, v=v, dout=d_out)
    # attn2d_o receive-buffer peaks per stream on a 3x3 grid (n=36, h=4): the
    # reference's double-buffering discipline (test_strategies.py:346-360)
    cfg = DistAttnConfig(n=36, h=4, p=9, mask=MaskKind.CAUSAL)
    q9, k9, v9, d9 = gen(36, 4, seed=36 * 31 + 9)
    fwd = run_forward("attn2d_o", cfg, q9, k9, v9)
    bwd = run_backward("attn2d_o", cfg, fwd.saved, d9)
    peaks = {}
    for src in (fwd.buffer_peaks, bwd.buffer_peaks):
        for (_, stream), pk in src.items():
            peaks[stream] = max(peaks.get(stream, 0), pk)
    streams = sorted(peaks)
    out.update(o_peaks_streams=np.array(streams), o_peaks=np.array([peaks[s] for s in streams]),
               o9_q=q9, o9_k=k9, o9_v=v9, o9_dout=d9, o9_o=fwd.o, o9_dq=bwd.dq, o9_dk=bwd.dk,
               o9_dv=bwd.dv)
    np.savez_compressed(OUT / "strategy_small.npz", **out)


def gpu_parity_cases():
    """bf16-rounded inputs, fp64 reference outputs, for the CUDA tile."""
    cases = [("n256_h64_causal", 256, 64, True, 1.0 / 8.0, 101),
             ("n256_h64_none_s1", 256, 64, False, 1.0, 102),
             ("n128_h128_causal", 128, 128, True, 1.0 / np.sqrt(128.0), 103),
             ("n320_h128_none", 320, 128, False, 1.0 / np.sqrt(128.0), 104)]
    out = {}
    for tag, n, h, causal, scale, seed in cases:
        q, k, v, d_out = (bf16_round(x) for x in gen(n, h, seed))
        idx = np.arange(n, dtype=np.int64)
        mask = MaskSpec.causal() if causal else MaskSpec.none()
        part = flash_attn_forward(TokenShard(q, idx), TokenShard(k, idx),
                                  TokenShard(v, idx), mask, scale, 64)
        o = finalize(part)
        dq, dk, dv = flash_attn_backward(TokenShard(q, idx), TokenShard(k, idx),
                                         TokenShard(v, idx), o, d_out, part.m, part.d,
                                         mask, scale)
        assert np.abs(o - reference_attention(q, k, v, mask, scale)).max() < 1e-12
        out.update({f"{tag}_q": bf16_bits(q), f"{tag}_k": bf16_bits(k),
                    f"{tag}_v": bf16_bits(v), f"{tag}_dout": bf16_bits(d_out),
                    f"{tag}_o": o.astype(np.float32),
                    f"{tag}_lse": part.logsumexp.astype(np.float32),
                    f"{tag}_dq": dq.astype(np.float32), f"{tag}_dk": dk.astype(np.float32),
                    f"{tag}_dv": dv.astype(np.float32),
                    f"{tag}_meta": np.array([n, h, int(causal), scale])})
        out[f"{tag}_pairs"] = np.array(count_unmasked(idx, idx, causal))
    np.savez_compressed(OUT / "gpu_parity.npz", **out)


def dropin_cases():
    """The reference's own attention-API test vectors on bf16-rounded inputs
    (so a bf16 kernel sees exactly the values the reference computed on),
    for the drop-in tests of the B200 path (tests/test_dropin.py):
    test_attention.py:123-157 (forward, index subsets, masked rows),
    :289-328 (backward, key-subset partial sums), test_kernels.py:124-137
    (streaming continuation), SPEC.md:132-133 (known answer), and the
    strategy entry points run_forward / run_backward at p in {1, 4}."""
    out = {}
    r = lambda seed, *shape: bf16_round(np.random.default_rng(seed).uniform(-1, 1, shape))  # noqa
    # forward vs blocks and masks (test_attention.py:123-130)
    q, k, v = r(40, 7, 4), r(41, 7, 4), r(42, 7, 4)
    out.update(fw_q=q, fw_k=k, fw_v=v)
    for mname, mask in (("none", MaskSpec.none()), ("causal", MaskSpec.causal())):
        for block in (1, 3, 64):
            part = flash_attn_forward(TokenShard(q, np.arange(7)), TokenShard(k, np.arange(7)),
                                      TokenShard(v, np.arange(7)), mask, 1.0, block)
            out[f"fw_{mname}_b{block}_o"] = finalize(part)
            out[f"fw_{mname}_b{block}_lse"] = part.logsumexp
    # index subsets (test_attention.py:136-145) and masked rows (:147-157)
    qi, ki = np.array([3, 9, 17]), np.array([2, 9, 12, 20])
    q, k, v = r(43, 3, 3), r(44, 4, 3), r(45, 4, 3)
    part = flash_attn_forward(TokenShard(q, qi), TokenShard(k, ki), TokenShard(v, ki),
                              MaskSpec.causal())
    out.update(sub_q=q, sub_k=k, sub_v=v, sub_qi=qi, sub_ki=ki, sub_o=finalize(part),
               sub_lse=part.logsumexp)
    q, k, v = r(46, 2, 2), r(47, 2, 2), r(48, 2, 2)
    part = flash_attn_forward(TokenShard(q, [0, 8]), TokenShard(k, [4, 5]),
                              TokenShard(v, [4, 5]), MaskSpec.causal())
    out.update(msk_q=q, msk_k=k, msk_v=v, msk_lse=part.logsumexp,
               msk_o1=part.n[1] / part.d[1])
    # streaming continuation (test_kernels.py:124-137), kernel level
    q, k, v, qi, ki = (bf16_round(x) if x.dtype == np.float64 else x
                       for x in random_problem(15))
    m = np.full(q.shape[0], -np.inf)
    nacc, d = np.zeros_like(q), np.zeros(q.shape[0])
    kernels.flash_forward(q, k, v, qi, ki, False, 1.0, 64, m, nacc, d)
    out.update(cont_q=q, cont_k=k, cont_v=v, cont_qi=qi, cont_ki=ki, cont_o=nacc / d[:, None],
               cont_lse=m + np.log(d))
    # backward full range (test_attention.py:289-300) and key-subset partial
    # sums (:302-328), both masks
    for mname, mask in (("none", MaskSpec.none()), ("causal", MaskSpec.causal())):
        n, h = 6, 3
        q, k, v, do = r(78, n, h), r(79, n, h), r(80, n, h), r(81, n, h)
        idx = np.arange(n)
        part = flash_attn_forward(TokenShard(q, idx), TokenShard(k, idx), TokenShard(v, idx),
                                  mask)
        o = finalize(part)
        dq, dk, dv = flash_attn_backward(TokenShard(q, idx), TokenShard(k, idx),
                                         TokenShard(v, idx), o, do, part.m, part.d, mask)
        out.update({f"bw_{mname}_{x}": y for x, y in
                    (("q", q), ("k", k), ("v", v), ("do", do), ("o", o), ("lse", part.logsumexp),
                     ("dq", dq), ("dk", dk), ("dv", dv))})
    # mid-size tile parity (h = 64 / 128, scale 1/sqrt(h)), kernel level
    for tag, n, h, causal, seed in (("mid_h64_causal", 256, 64, True, 201),
                                    ("mid_h128_none", 256, 128, False, 202)):
        q, k, v, do = (bf16_round(x) for x in gen(n, h, seed))
        idx = np.arange(n)
        mask = MaskSpec.causal() if causal else MaskSpec.none()
        sc = 1.0 / np.sqrt(h)
        part = flash_attn_forward(TokenShard(q, idx), TokenShard(k, idx), TokenShard(v, idx),
                                  mask, sc)
        o = finalize(part)
        dq, dk, dv = flash_attn_backward(TokenShard(q, idx), TokenShard(k, idx),
                                         TokenShard(v, idx), o, do, part.m, part.d, mask, sc)
        out.update({f"{tag}_{x}": y for x, y in
                    (("q", q), ("k", k), ("v", v), ("do", do), ("o", o), ("lse", part.logsumexp),
                     ("dq", dq), ("dk", dk), ("dv", dv))})
        out[f"{tag}_meta"] = np.array([n, h, int(causal), sc])
    # strategy entry points (strategies/__init__.py:40-46) on the simulated grid
    for name in ("attn2d_no", "attn2d_o", "ring"):
        for p in (1, 4):
            for causal in (False, True):
                n, h = 64, 8
                mask = MaskKind.CAUSAL if causal else MaskKind.NONE
                cfg = DistAttnConfig(n=n, h=h, p=p, mask=mask, scale=h ** -0.5)
                q, k, v, do = (bf16_round(x) for x in gen(n, h, seed=700 + p))
                fwd = run_forward(name, cfg, q, k, v)
                bwd = run_backward(name, cfg, fwd.saved, do)
                tag = f"st_{name}_p{p}_{'causal' if causal else 'none'}"
                out.update({f"{tag}_o": fwd.o, f"{tag}_dq": bwd.dq, f"{tag}_dk": bwd.dk,
                            f"{tag}_dv": bwd.dv})
                out[f"st_in_p{p}"] = np.stack([q, k, v, do])
    # fp32 storage: inputs are bf16 values (exact), outputs far more precise
    # than the bf16-kernel tolerance they are checked at
    out = {k: (v.astype(np.float32) if v.dtype == np.float64 else v) for k, v in out.items()}
    np.savez_compressed(OUT / "dropin.npz", **out)


if __name__ == "__main__":
    only = sys.argv[1:]
    for fn in (tile_cases, merge_cases, strategy_cases, gpu_parity_cases, dropin_cases):
        if not only or fn.__name__ in only:
            fn()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
