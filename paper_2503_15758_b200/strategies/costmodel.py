"""Exact per-rank communication identities of this package's schedules and a
reconcile report against the measured ledger.

The B200 counterpart of the reference's exact schedule counts
(`costmodel.predicted_phase_words` / `predicted_phase_msgs`,
pkg/src/attn2d/costmodel.py:106-153) and of `reconcile` (:307-325),
generalised from square p = s^2 grids to Pr x Pc and to the forms this
package moves:

* partial results are (O, LSE): h + 1 words per row instead of the
  reference's (m, n, d) = h + 2;
* the backward row bundle is (Q, dO, LSE, delta): 2h + 2 words instead of
  the reference's (q, o, d_out, m, d) = 3h + 2 (delta = rowsum(dO * O) is
  computed by the owner before the gather);
* words are counted per element AND as bytes, because the dtypes differ per
  op (bf16 Q/K/V/dO, fp32 partials, statistics and gradient reductions);
* a collective over n ranks counts n - 1 messages (the relay hops the
  reference's mesh counts); K and V, O and LSE travel as separate
  collectives in attn2d_no, and every head chunk repeats its collectives.

For a square grid with one head the attn2d_o schedule reproduces the
reference's message counts exactly and its word counts up to the two form
differences above (tests/test_costmodel.py checks both against the
reference's own formula).
"""

from __future__ import annotations

from dataclasses import dataclass

from ..errors import ConfigError
from ..layouts import Grid2D
from .attn2d_no import _chunks

PHASE_FWD, PHASE_BWD = "attention_fwd", "attention_bwd"
BF16, F32 = 2, 4
SIMULATED = ("attn2d_no", "attn2d_o", "ring")


@dataclass(frozen=True)
class OpTraffic:
    words: int
    bytes: int
    msgs: int


def _op(words: int, width: int, msgs: int) -> OpTraffic:
    return OpTraffic(int(words), int(words) * width, int(msgs))


def predicted_ops(strategy: str, n: int, h: int, heads: int, grid: Grid2D, rank: int,
                  phase: str, head_chunks: int = 1) -> dict[str, OpTraffic]:
    """Traffic one rank sends during one phase, by ledger op name."""
    if strategy not in SIMULATED:
        raise ConfigError(f"no exact schedule counts for strategy {strategy!r}")
    if phase not in (PHASE_FWD, PHASE_BWD):
        raise ConfigError(f"phase must be {PHASE_FWD!r} or {PHASE_BWD!r}, got {phase!r}")
    P = grid.p
    if n % P:
        raise ConfigError(f"p={P} must divide n={n}")
    L, B = n // P, heads
    out: dict[str, OpTraffic] = {}
    if strategy == "ring":
        if P == 1:
            return out
        out["ring_kv"] = _op(2 * (P - 1) * L * B * h, BF16, P - 1)
        if phase == PHASE_BWD:
            out["ring_kvg"] = _op(2 * (P - 1) * L * B * h, F32, P - 1)
            out["ring_home"] = _op(2 * L * B * h, F32, 1)
        return out
    pr, pc = grid.pr, grid.pc
    r, c = grid.coord(rank)
    off_diag = grid.kv_dest(r, c) != rank
    nch = len(_chunks(B, head_chunks)) if strategy == "attn2d_no" else 1
    if phase == PHASE_FWD:
        if off_diag:
            out["transpose_kv"] = _op(2 * L * B * h, BF16, 1)
        if strategy == "attn2d_no":
            if pc > 1:
                out["gather_q"] = _op((pc - 1) * L * B * h, BF16, (pc - 1) * nch)
                out["merge_partials"] = _op((pc - 1) * L * B * (h + 1), F32, 2 * (pc - 1) * nch)
            if pr > 1:
                out["gather_kv"] = _op(2 * (pr - 1) * L * B * h, BF16, 2 * (pr - 1) * nch)
        else:
            if pc > 1:
                out["forward_q"] = _op((pc - 1) * L * B * h, BF16, pc - 1)
                out["scatter_partial"] = _op((pc - 1) * L * B * (h + 1), F32, pc - 1)
            if pr > 1:
                out["gather_kv"] = _op(2 * (pr - 1) * L * B * h, BF16, pr - 1)
        return out
    bundle_words = (pc - 1) * L * B * (2 * h + 2)
    bundle_bytes = (pc - 1) * L * B * (2 * h * BF16 + 2 * F32)
    if strategy == "attn2d_no":
        if pc > 1:
            out["bwd_gather_row"] = OpTraffic(bundle_words, bundle_bytes, 3 * (pc - 1) * nch)
            out["rs_dq"] = _op((pc - 1) * L * B * h, F32, (pc - 1) * nch)
        if pr > 1:
            out["bwd_gather_kv"] = _op(2 * (pr - 1) * L * B * h, BF16, 2 * (pr - 1) * nch)
            out["rs_dkv"] = _op(2 * (pr - 1) * L * B * h, F32, 2 * (pr - 1) * nch)
        if off_diag:  # reduced dK/dV return in fp32 when they were reduced, else bf16
            out["transpose_dkv"] = _op(2 * L * B * h, F32 if pr > 1 else BF16, 1)
        return out
    if pc > 1:
        out["forward_qod"] = OpTraffic(bundle_words, bundle_bytes, pc - 1)
        out["scatter_dq"] = _op((pc - 1) * L * B * h, F32, pc - 1)
    if pr > 1:
        out["gather_kv"] = _op(2 * (pr - 1) * L * B * h, BF16, pr - 1)
        # ring reduction up the column (one message per hop), or two
        # reduce-scatters when the grid has a single column
        out["scatter_dkv"] = _op(2 * (pr - 1) * L * B * h, F32,
                                 (pr - 1) if pc > 1 else 2 * (pr - 1))
    if off_diag:
        out["transpose_dkv"] = _op(2 * L * B * h, F32, 1)
    return out


def predicted_phase_words(strategy, n, h, heads, grid, rank, phase, head_chunks=1) -> int:
    return sum(t.words for t in predicted_ops(strategy, n, h, heads, grid, rank, phase,
                                              head_chunks).values())


def predicted_phase_msgs(strategy, n, h, heads, grid, rank, phase, head_chunks=1) -> int:
    return sum(t.msgs for t in predicted_ops(strategy, n, h, heads, grid, rank, phase,
                                             head_chunks).values())


@dataclass(frozen=True)
class ReconcileRow:
    rank: int
    phase: str
    op: str
    measured: OpTraffic
    predicted: OpTraffic

    @property
    def match(self) -> bool:
        return self.measured == self.predicted


@dataclass(frozen=True)
class ReconcileReport:
    strategy: str
    rows: tuple

    @property
    def ok(self) -> bool:
        return all(r.match for r in self.rows)

    def mismatches(self) -> list:
        return [r for r in self.rows if not r.match]


def reconcile(ledger, strategy: str, n: int, h: int, heads: int, grid: Grid2D, rank: int,
              head_chunks: int = 1, phases=(PHASE_FWD, PHASE_BWD)) -> ReconcileReport:
    """Measured (strategies.comm.ByteLedger) against predicted traffic of one
    rank, op by op and phase by phase (reference costmodel.py:307-325)."""
    rows = []
    for phase in phases:
        pred = predicted_ops(strategy, n, h, heads, grid, rank, phase, head_chunks)
        meas = {op: OpTraffic(v[3], v[0], v[4]) for (ph, op), v in ledger.rows.items()
                if ph == phase}
        for op in sorted(set(pred) | set(meas)):
            rows.append(ReconcileRow(rank, phase, op, meas.get(op, OpTraffic(0, 0, 0)),
                                     pred.get(op, OpTraffic(0, 0, 0))))
    return ReconcileReport(strategy, tuple(rows))
