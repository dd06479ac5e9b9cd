"""Per-tensor error report of the B200 path against the reference (north_star:
"max-abs and relative error reported for O, LSE, dQ, dK and dV").

    python tools/parity_report.py [--out profiles/parity.json] [--quick]

Inputs follow SURVEY.md §8c's parity protocol: uniform[-1, 1] values (numpy
default_rng for C1, torch.Generator for the GPU sizes), rounded ONCE to bf16,
the same rounded values fed to both sides.  The reference side is the
UNMODIFIED reference package (pip-installed in baseline/_ref, numpy kernel
backend, float64); if it is not importable the oracle port
(oracle/attn2d_oracle.py, the same numpy recurrences) stands in and the
report says so.  The B200 side is the product path: functional-level tile
forward (bf16 O + fp32 LSE) and backward (bf16 dQ, dK, dV).

Configs (BASELINE.json):
  C1      B=1, M=4, N=2048, H=64, non-causal, scale 1/sqrt(H): every element
          of every head; the reference runs its attn2d_no strategy on the
          simulated 2x2 grid (run_forward / run_backward) and its streaming
          kernel for the LSE.
  C2      B=1, M=32, N=32768, H=128, causal: head 0, row-sampled O / LSE / dQ
          (512 rows against all keys) and key-sampled dK / dV (512 keys
          against all queries, global statistics from the reference's own
          streaming forward over all rows).
  metric  B=1, M=32, N=131072, H=128, causal: head 0, row-sampled O / LSE /
          dQ through the reference; key-sampled dK / dV through the
          reference's flash_attn_backward with the global row statistics and
          O computed in fp64 on the GPU (a full reference forward at this
          size takes hours on the host).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF = ROOT / "baseline" / "_ref"
CALIBRATION = {"rel_fro": 2.3e-3, "lse_max_abs": 1e-6,
               "source": "SURVEY.md §8c: ideal bf16-P / fp32-accumulate kernel vs fp64"}
GATE = {"rel_fro": 1e-2, "lse_max_abs": 1e-3}


def reference_api():
    """(flash_attn_forward, flash_attn_backward, finalize, TokenShard, MaskSpec,
    run_forward, run_backward, DistAttnConfig, MaskKind, kind)."""
    if (REF / "attn2d").is_dir():
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/a2d_numba_cache")
        os.environ["ATTN2D_KERNEL"] = "numpy"
        sys.path.insert(0, str(REF))
        from attn2d import kernels
        from attn2d.attention import (MaskKind, MaskSpec, TokenShard, finalize,
                                      flash_attn_backward, flash_attn_forward)
        from attn2d.strategies import DistAttnConfig, run_backward, run_forward
        kernels.use_backend("numpy")

        def fwd(q, k, v, qi, ki, causal, scale):
            part = flash_attn_forward(TokenShard(q, qi), TokenShard(k, ki), TokenShard(v, ki),
                                      MaskSpec.causal() if causal else MaskSpec.none(), scale)
            return finalize(part), part.logsumexp, (part.m, part.d)

        def bwd(q, k, v, o, do, md, qi, ki, causal, scale):
            return flash_attn_backward(TokenShard(q, qi), TokenShard(k, ki), TokenShard(v, ki),
                                       o, do, md[0], md[1],
                                       MaskSpec.causal() if causal else MaskSpec.none(), scale)

        def strat(q, k, v, do, causal, scale, p=4):
            cfg = DistAttnConfig(n=q.shape[0], h=q.shape[1], p=p,
                                 mask=MaskKind.CAUSAL if causal else MaskKind.NONE, scale=scale)
            f = run_forward("attn2d_no", cfg, q, k, v)
            b = run_backward("attn2d_no", cfg, f.saved, do)
            return f.o, b.dq, b.dk, b.dv

        return fwd, bwd, strat, "reference (baseline/_ref attn2d 0.1.0, numpy backend, fp64)"
    from oracle import attn2d_oracle as orc

    def fwd(q, k, v, qi, ki, causal, scale):
        o, lse, md = orc.tile_forward_full(q, k, v, qi, ki, causal, scale)
        return o, lse, md

    def bwd(q, k, v, o, do, md, qi, ki, causal, scale):
        return orc.tile_backward_full(q, k, v, o, do, md[0], md[1], qi, ki, causal, scale)

    return fwd, bwd, None, "oracle port (oracle/attn2d_oracle.py; reference not installed)"


def errs(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    fin = np.isfinite(want)
    d = np.abs(got[fin] - want[fin])
    return {"max_abs": float(d.max()), "rel_fro":
            float(np.linalg.norm(got[fin] - want[fin]) / max(np.linalg.norm(want[fin]), 1e-300)),
            "ref_max_abs": float(np.abs(want[fin]).max()), "elements": int(fin.sum())}


def b200_fwd_bwd(q, k, v, do, causal, scale):
    """Product path on [bh, n, h] bf16 CUDA tensors: O (bf16), LSE, dQ/dK/dV (bf16)."""
    from paper_2503_15758_b200 import functional, ops
    o, lse = ops.tile_forward(q, k, v, causal=causal, scale=scale, out_dtype=torch.bfloat16)
    dq, dk, dv = functional.attention_backward(q, k, v, o, lse, do, causal, scale)
    torch.cuda.synchronize()
    return o, lse, dq, dk, dv


def c1(fwd, bwd, strat):
    n, h, m, causal = 2048, 64, 4, False
    scale = h ** -0.5
    rng = np.random.default_rng(0)
    x = [rng.uniform(-1, 1, (m, n, h)) for _ in range(4)]
    xb = [torch.tensor(a).to(torch.bfloat16) for a in x]
    q, k, v, do = (t.double().numpy() for t in xb)
    o, lse, dq, dk, dv = (t.double().cpu().numpy() for t in
                          b200_fwd_bwd(*(t.cuda() for t in xb), causal, scale))
    want = {x: [] for x in ("O", "LSE", "dQ", "dK", "dV")}
    idx = np.arange(n)
    t0 = time.perf_counter()
    for b in range(m):
        ro, rlse, md = fwd(q[b], k[b], v[b], idx, idx, causal, scale)
        if strat is not None:  # the 2x2 simulated-grid strategy (C1 as BASELINE.json states)
            so, sdq, sdk, sdv = strat(q[b], k[b], v[b], do[b], causal, scale)
            assert np.abs(so - ro).max() < 1e-10
        else:
            sdq, sdk, sdv = bwd(q[b], k[b], v[b], ro, do[b], md, idx, idx, causal, scale)
            so = ro
        for key, val in zip(("O", "LSE", "dQ", "dK", "dV"), (so, rlse, sdq, sdk, sdv)):
            want[key].append(val)
    secs = time.perf_counter() - t0
    got = {"O": o, "LSE": lse, "dQ": dq, "dK": dk, "dV": dv}
    return {"shape": "B=1 M=4 N=2048 H=64 non-causal scale=1/sqrt(H)",
            "sampling": "all elements, all 4 heads" +
                        ("; reference = run_forward/run_backward('attn2d_no', p=4)"
                         if strat is not None else ""),
            "reference_seconds": secs,
            "errors": {key: errs(got[key], np.stack(want[key])) for key in got}}


def sampled(fwd, bwd, n, bh, samples, full_stats_on_host, seed=0):
    h, causal = 128, True
    scale = h ** -0.5
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v, do = (torch.empty((bh, n, h), dtype=torch.bfloat16, device="cuda")
                   .uniform_(-1, 1, generator=g) for _ in range(4))
    o, lse, dq, dk, dv = b200_fwd_bwd(q, k, v, do, causal, scale)
    b = 0
    qh, kh, vh, doh = (t[b].double().cpu().numpy() for t in (q, k, v, do))
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(n, samples, replace=False)).astype(np.int64)
    keys = np.sort(rng.choice(n, samples, replace=False)).astype(np.int64)
    idx = np.arange(n, dtype=np.int64)
    t0 = time.perf_counter()
    ro, rlse, md = fwd(qh[rows], kh, vh, rows, idx, causal, scale)
    rdq, _, _ = bwd(qh[rows], kh, vh, ro, doh[rows], md, rows, idx, causal, scale)
    if full_stats_on_host:
        fo, _, fmd = fwd(qh, kh, vh, idx, idx, causal, scale)
        stats = "reference streaming forward over all rows"
    else:  # fp64 on the GPU, chunked over rows
        kk, vv = k[b].double(), v[b].double()
        fo = np.empty((n, h))
        fm = np.empty(n)
        for r0 in range(0, n, 4096):
            qq = q[b, r0:r0 + 4096].double()
            s = (qq @ kk.T) * scale
            qi = torch.arange(r0, r0 + qq.shape[0], device="cuda")
            s.masked_fill_(qi[:, None] < torch.arange(n, device="cuda")[None, :], float("-inf"))
            mx = s.max(1).values
            pexp = torch.exp(s - mx[:, None])
            dsum = pexp.sum(1)
            fo[r0:r0 + qq.shape[0]] = ((pexp @ vv) / dsum[:, None]).cpu().numpy()
            fm[r0:r0 + qq.shape[0]] = (mx + torch.log(dsum)).cpu().numpy()
            del s, pexp
        fmd = (fm, np.ones(n))  # (m, d) = (LSE, 1): the same statistics
        stats = "global row statistics and O in fp64 on the GPU (chunked)"
    _, rdk, rdv = bwd(qh, kh[keys], vh[keys], fo, doh, fmd, idx, keys, causal, scale)
    secs = time.perf_counter() - t0
    got = {"O": o[b, rows], "LSE": lse[b, rows], "dQ": dq[b, rows], "dK": dk[b, keys],
           "dV": dv[b, keys]}
    want = {"O": ro, "LSE": rlse, "dQ": rdq, "dK": rdk, "dV": rdv}
    return {"shape": f"B=1 M={bh} N={n} H=128 causal scale=1/sqrt(H) (head 0 checked)",
            "sampling": f"{samples} random rows (O, LSE, dQ) and {samples} random keys (dK, dV) "
                        f"of head 0; dK/dV statistics: {stats}",
            "reference_seconds": secs,
            "errors": {key: errs(got[key].double().cpu().numpy(), want[key]) for key in got}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "parity.json"))
    ap.add_argument("--quick", action="store_true", help="C1 only")
    args = ap.parse_args()
    fwd, bwd, strat, kind = reference_api()
    try:
        commit = subprocess.run(["git", "rev-parse", "--short", "HEAD"], cwd=ROOT,
                                capture_output=True, text=True).stdout.strip() or None
    except OSError:
        commit = None
    rep = {"reference": kind, "calibration": CALIBRATION, "gate": GATE,
           "gpu": torch.cuda.get_device_name(0), "commit": commit,
           "outputs": "product dtypes: O, dQ, dK, dV bf16; LSE fp32", "configs": {}}
    rep["configs"]["C1"] = c1(fwd, bwd, strat)
    print(json.dumps({"C1": rep["configs"]["C1"]["errors"]}), flush=True)
    if not args.quick:
        rep["configs"]["C2"] = sampled(fwd, bwd, 32768, 32, 512, True)
        print(json.dumps({"C2": rep["configs"]["C2"]["errors"]}), flush=True)
        rep["configs"]["metric"] = sampled(fwd, bwd, 131072, 32, 256, False)
        print(json.dumps({"metric": rep["configs"]["metric"]["errors"]}), flush=True)
    worst = {}
    for cfg in rep["configs"].values():
        for key, e in cfg["errors"].items():
            m = "lse_max_abs" if key == "LSE" else "rel_fro"
            v = e["max_abs"] if key == "LSE" else e["rel_fro"]
            worst[key] = max(worst.get(key, 0.0), v)
            cfg.setdefault("within_gate", True)
            cfg["within_gate"] = cfg["within_gate"] and v <= GATE[m]
    rep["worst"] = worst
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(rep, indent=1))
    print("wrote", args.out)


if __name__ == "__main__":
    main()
