"""Grid communication over torch.distributed (NCCL over NVLink on the B200
box; gloo in the CPU tests) — the B200 replacement of the reference's
simulated Proc endpoint (pkg/src/attn2d/mesh.py:308-408):

  reference                          here
  send_recv (transpose_kv)           permute()            batch_isend_irecv
  all_gather (row / column)          row/col_all_gather() all_gather_into_tensor
  reduce_scatter(attn_fix)           row_all_to_all() + the LSE-merge kernel
  reduce_scatter(sum)                row/col_reduce_scatter() reduce_scatter_tensor (fp32)

Every call charges a per-rank byte ledger (the reference's CommLedger,
mesh.py:106-191) with the logical payload that leaves the rank, so the
volume identities of costmodel.predicted_phase_words (costmodel.py:106-136)
can be checked on real transfers.
"""

from __future__ import annotations

from collections import defaultdict
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from ..layouts import Grid2D


@dataclass
class ByteLedger:
    """Per-rank traffic by (phase, op): bytes out / in, API calls, words
    (elements) out and point-to-point messages out.  A collective over n
    ranks counts n - 1 messages (the relay hops of the reference's
    mesh.py:106-191 ledger); a send to one peer counts 1."""

    rows: dict = field(default_factory=lambda: defaultdict(lambda: [0, 0, 0, 0, 0]))

    def charge(self, phase: str, op: str, bytes_out: int, bytes_in: int, words_out: int = 0,
               msgs_out: int = 1):
        row = self.rows[(phase, op)]
        row[0] += int(bytes_out)
        row[1] += int(bytes_in)
        row[2] += 1
        row[3] += int(words_out)
        row[4] += int(msgs_out)

    def bytes_out(self, phase: str | None = None) -> int:
        return sum(v[0] for (ph, _), v in self.rows.items() if phase in (None, ph))

    def words_out(self, phase: str | None = None) -> int:
        return sum(v[3] for (ph, _), v in self.rows.items() if phase in (None, ph))

    def msgs_out(self, phase: str | None = None) -> int:
        return sum(v[4] for (ph, _), v in self.rows.items() if phase in (None, ph))

    def as_dict(self) -> dict:
        return {f"{ph}/{op}": {"bytes_out": v[0], "bytes_in": v[1], "calls": v[2],
                               "words_out": v[3], "msgs_out": v[4]}
                for (ph, op), v in sorted(self.rows.items())}


def _nbytes(t: torch.Tensor) -> int:
    return t.numel() * t.element_size()


class GridComm:
    """Row / column process groups of a Pr x Pc grid laid over the world."""

    def __init__(self, grid: Grid2D, group=None):
        self.grid = grid
        self.world = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        size = dist.get_world_size(group) if dist.is_initialized() else 1
        if size != grid.p:
            raise ValueError(f"world size {size} != grid {grid.pr}x{grid.pc}")
        self.r, self.c = grid.coord(self.rank)
        self.row_group = self.col_group = None
        if grid.p > 1:
            # every rank must create every group, in the same order
            for r in range(grid.pr):
                g = dist.new_group(grid.row_ranks(r))
                if r == self.r:
                    self.row_group = g
            for c in range(grid.pc):
                g = dist.new_group(grid.col_ranks(c))
                if c == self.c:
                    self.col_group = g
        self.ledger = ByteLedger()
        self.phase = "attention_fwd"
        # live receive buffers per stream (the reference's buffer accounting,
        # mesh.py:455-475): opened when a receive is posted, closed when the
        # schedule releases the buffer
        self.buffer_peaks: dict = {}
        self._live: dict = defaultdict(int)

    def buf_open(self, stream: str):
        self._live[stream] += 1
        self.buffer_peaks[stream] = max(self.buffer_peaks.get(stream, 0), self._live[stream])

    def buf_close(self, stream: str):
        self._live[stream] -= 1

    # ------------------------------------------------------------ helpers
    def _gather(self, t: torch.Tensor, group, n: int, op: str, async_op=False):
        if n == 1:
            return (t, None) if async_op else t
        out = torch.empty((n * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        work = dist.all_gather_into_tensor(out, t.contiguous(), group=group, async_op=async_op)
        self.ledger.charge(self.phase, op, _nbytes(t) * (n - 1), _nbytes(t) * (n - 1),
                           t.numel() * (n - 1), n - 1)
        return (out, work) if async_op else out

    def row_all_gather(self, t, op="gather_q", async_op=False):
        return self._gather(t, self.row_group, self.grid.pc, op, async_op)

    def col_all_gather(self, t, op="gather_kv", async_op=False):
        return self._gather(t, self.col_group, self.grid.pr, op, async_op)

    def _reduce_scatter(self, t: torch.Tensor, group, n: int, op: str, async_op=False):
        if n == 1:
            return (t, None) if async_op else t
        out = torch.empty((t.shape[0] // n,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        t = t.contiguous()
        self.ledger.charge(self.phase, op, _nbytes(out) * (n - 1), _nbytes(out) * (n - 1),
                           out.numel() * (n - 1), n - 1)
        if dist.get_backend(group) == "gloo":
            # gloo has no reduce_scatter: all_reduce and keep this rank's chunk
            work = dist.all_reduce(t, group=group)
            out.copy_(t.chunk(n, 0)[dist.get_rank(group)])
            return (out, None) if async_op else out
        work = dist.reduce_scatter_tensor(out, t, op=dist.ReduceOp.SUM, group=group,
                                          async_op=async_op)
        return (out, work) if async_op else out

    def row_reduce_scatter(self, t, op="rs_dq", async_op=False):
        return self._reduce_scatter(t, self.row_group, self.grid.pc, op, async_op)

    def col_reduce_scatter(self, t, op="rs_dkv", async_op=False):
        return self._reduce_scatter(t, self.col_group, self.grid.pr, op, async_op)

    def row_all_to_all(self, t: torch.Tensor, op="merge_partials", async_op=False):
        n = self.grid.pc
        if n == 1:
            return (t, None) if async_op else t
        t = t.contiguous()
        out = torch.empty_like(t)
        self.ledger.charge(self.phase, op, _nbytes(t) // n * (n - 1), _nbytes(t) // n * (n - 1),
                           t.numel() // n * (n - 1), n - 1)
        work = dist.all_to_all_single(out, t, group=self.row_group, async_op=async_op)
        return (out, work) if async_op else out

    def exchange(self, sends: list[torch.Tensor], dst: int, src: int, op: str, async_op=False,
                 recv_into: list[torch.Tensor] | None = None):
        """Send `sends` to world rank dst and receive same-shaped tensors from src
        (the reference's send_recv, mesh.py:308-323), optionally straight into
        caller-provided (contiguous) buffers."""
        if dst == self.rank and src == self.rank:
            if recv_into is not None:
                for b, t in zip(recv_into, sends):
                    b.copy_(t)
                return (list(recv_into), None) if async_op else list(recv_into)
            return (list(sends), None) if async_op else list(sends)
        recvs = list(recv_into) if recv_into is not None else [torch.empty_like(t) for t in sends]
        ops = [dist.P2POp(dist.isend, t.contiguous(), dst) for t in sends]
        ops += [dist.P2POp(dist.irecv, b, src) for b in recvs]
        reqs = dist.batch_isend_irecv(ops)
        nb = sum(_nbytes(t) for t in sends)
        self.ledger.charge(self.phase, op, nb, nb, sum(t.numel() for t in sends), 1)
        if async_op:
            return recvs, reqs
        for q in reqs:
            q.wait()
        return recvs

    def permute_kv(self, k, v, async_op=False):
        g = self.grid
        return self.exchange([k, v], g.kv_dest(self.r, self.c), g.kv_src(self.r, self.c),
                             "transpose_kv", async_op)

    def unpermute_kv(self, dk, dv, async_op=False):
        g = self.grid
        return self.exchange([dk, dv], g.kv_src(self.r, self.c), g.kv_dest(self.r, self.c),
                             "transpose_dkv", async_op)


def wait_all(work):
    if work is None:
        return
    if isinstance(work, (list, tuple)):
        for w in work:
            wait_all(w)
        return
    work.wait()
