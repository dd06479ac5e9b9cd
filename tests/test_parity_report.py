"""The per-tensor error report (tools/parity_report.py) at C1 — B=1, M=4,
N=2048, H=64, non-causal, every element of every head, the reference's
attn2d_no strategy on its simulated 2x2 grid — must stay inside the gate
(rel-Fro <= 1e-2 on O/dQ/dK/dV, LSE max-abs <= 1e-3) and
report finite, non-zero errors (a zero error would mean the kernels did not
run in bf16)."""

import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_c1_error_report_within_gate():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, str(ROOT / "tools"))
    import parity_report as pr
    fwd, bwd, strat, kind = pr.reference_api()
    rep = pr.c1(fwd, bwd, strat)
    print(kind, rep["errors"])
    for key, e in rep["errors"].items():
        if key == "LSE":
            assert e["max_abs"] <= pr.GATE["lse_max_abs"], (key, e)
        else:
            assert 0.0 < e["rel_fro"] <= pr.GATE["rel_fro"], (key, e)
