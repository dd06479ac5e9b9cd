"""Attention2D, non-overlapped schedule (reference strategies/attn2d_no.py;
PAPER Alg. 1 forward, Alg. 3 backward) on a Pr x Pc grid of B200s.

Forward on rank (r, c), local shards [L, BH, H] (token-major, L = N/P):
  1. permute K/V to the row-major residue (the mirror transpose, :81-82);
  2. all-gather Q along the grid row, K/V along the grid column (:85-89) —
     gathered buffers stay in all-gather order; the tile kernel reads their
     global indices from affine-blocked maps, so no re-sort is needed (the
     reference argsorts, :31-37);
  3. tile forward on (Q_g(r), K_g(c)) -> partial (O fp32, LSE) (:92-94);
  4. merge across the row: all_to_all of the partial slices (this rank's
     query rows are block c of Q_g) + one Pc-way LSE-merge kernel — the
     reduce-scatter with attn_fix of :44-57, with finalize fused (:97).
Backward (:116-167): all-gather (Q, dO, LSE, delta) along the row and K/V
along the column, tile backward, reduce-scatter dQ along the row and dK/dV
along the column (fp32 sums), inverse permutation of dK/dV.

Communication is overlapped with compute by head-chunk pipelining: the
gathers of chunk i+1 and the merge exchange of chunk i-1 are in flight
(NCCL streams) while chunk i's tile runs on the compute stream.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .. import ops as _ops
from ..layouts import Grid2D
from .comm import GridComm, wait_all


@dataclass
class Saved2D:
    """Exactly what a rank keeps from forward for backward (common.py:64-80):
    its query shard, the permuted key/value shard, its output and the global
    LSE of its query rows."""

    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    o: torch.Tensor
    lse: torch.Tensor  # [L, BH] fp32

    @property
    def words(self) -> int:
        return int(self.q.numel() + self.k.numel() + self.v.numel() + self.o.numel()
                   + self.lse.numel())


def _heads(t: torch.Tensor) -> torch.Tensor:
    """[rows, BH, H] token-major -> [BH, rows, H] view for the kernels."""
    return t.transpose(0, 1)


def _chunks(bh: int, n: int):
    n = max(1, min(n, bh))
    step = -(-bh // n)
    return [(i, min(i + step, bh)) for i in range(0, bh, step)]


class Attention2D:
    def __init__(self, comm: GridComm, n: int, causal: bool, scale: float, head_chunks: int = 1,
                 compute=None):
        self.comm = comm
        self.grid: Grid2D = comm.grid
        self.n = n
        self.L = self.grid.check_n(n)
        self.causal = bool(causal)
        self.scale = float(scale)
        self.head_chunks = head_chunks
        self.ops = compute if compute is not None else _ops
        self.q_index = self.grid.q_gathered(n, comm.r)
        self.k_index = self.grid.k_gathered(n, comm.c)

    # ------------------------------------------------------------------ fwd
    def _tile_fwd(self, q_g, k_g, v_g):
        g, L = self.grid, self.L
        bh, h = q_g.shape[1], q_g.shape[2]
        if g.pc == 1:
            o = torch.empty((L, bh, h), dtype=q_g.dtype, device=q_g.device)
            lse = torch.empty((bh, L), dtype=torch.float32, device=q_g.device)
            self.ops.tile_forward(_heads(q_g), _heads(k_g), _heads(v_g), causal=self.causal,
                                  scale=self.scale, q_index=self.q_index, k_index=self.k_index,
                                  out=_heads(o), lse=lse, out_dtype=q_g.dtype)
            return o, lse.t().contiguous()
        o_part = torch.empty((g.pc * L, bh, h), dtype=torch.float32, device=q_g.device)
        lse_part = torch.empty((bh, g.pc * L), dtype=torch.float32, device=q_g.device)
        self.ops.tile_forward(_heads(q_g), _heads(k_g), _heads(v_g), causal=self.causal,
                              scale=self.scale, q_index=self.q_index, k_index=self.k_index,
                              out=_heads(o_part), lse=lse_part)
        return o_part, lse_part.t().contiguous()

    def _merge(self, recv_o, recv_lse, dtype):
        g, L = self.grid, self.L
        bh, h = recv_o.shape[1], recv_o.shape[2]
        o, lse = self.ops.lse_merge(recv_o.view(g.pc, L * bh, h), recv_lse.view(g.pc, L * bh),
                                    out_dtype=dtype)
        return o.view(L, bh, h), lse.view(L, bh)

    def forward(self, q_p: torch.Tensor, k_p: torch.Tensor, v_p: torch.Tensor):
        comm, g = self.comm, self.grid
        comm.phase = "attention_fwd"
        k_t, v_t = comm.permute_kv(k_p, v_p)
        chunks = _chunks(q_p.shape[1], self.head_chunks)

        def gathers(i):
            a, b = chunks[i]
            sl = slice(a, b)
            q_g, w1 = comm.row_all_gather(q_p[:, sl].contiguous(), async_op=True)
            k_g, w2 = comm.col_all_gather(k_t[:, sl].contiguous(), async_op=True)
            v_g, w3 = comm.col_all_gather(v_t[:, sl].contiguous(), async_op=True)
            return (q_g, k_g, v_g), (w1, w2, w3)

        outs_o, outs_lse = [None] * len(chunks), [None] * len(chunks)
        pending = None  # (chunk, recv_o, recv_lse, work)
        nxt = gathers(0)
        for i in range(len(chunks)):
            cur = nxt
            if i + 1 < len(chunks):
                nxt = gathers(i + 1)
            wait_all(cur[1])
            o_i, lse_i = self._tile_fwd(*cur[0])
            if g.pc == 1:
                outs_o[i], outs_lse[i] = o_i, lse_i
                continue
            ro, w1 = comm.row_all_to_all(o_i, async_op=True)
            rl, w2 = comm.row_all_to_all(lse_i, async_op=True)
            if pending is not None:
                j, po, pl, pw = pending
                wait_all(pw)
                outs_o[j], outs_lse[j] = self._merge(po, pl, q_p.dtype)
            pending = (i, ro, rl, (w1, w2))
        if pending is not None:
            j, po, pl, pw = pending
            wait_all(pw)
            outs_o[j], outs_lse[j] = self._merge(po, pl, q_p.dtype)
        o_p = outs_o[0] if len(chunks) == 1 else torch.cat(outs_o, dim=1)
        lse_p = outs_lse[0] if len(chunks) == 1 else torch.cat(outs_lse, dim=1)
        return o_p, Saved2D(q=q_p, k=k_t, v=v_t, o=o_p, lse=lse_p)

    # ------------------------------------------------------------------ bwd
    def backward(self, saved: Saved2D, do_p: torch.Tensor):
        comm, g, L = self.comm, self.grid, self.L
        comm.phase = "attention_bwd"
        bh_all, h = do_p.shape[1], do_p.shape[2]
        delta = self.ops.bwd_preprocess(_heads(saved.o), _heads(do_p))      # [BH, L]
        stats = torch.stack([saved.lse, delta.t()], dim=-1).contiguous()    # [L, BH, 2]
        chunks = _chunks(bh_all, self.head_chunks)

        def gathers(i):
            a, b = chunks[i]
            sl = slice(a, b)
            q_g, w1 = comm.row_all_gather(saved.q[:, sl].contiguous(), "bwd_gather_row", True)
            do_g, w2 = comm.row_all_gather(do_p[:, sl].contiguous(), "bwd_gather_row", True)
            st_g, w3 = comm.row_all_gather(stats[:, sl].contiguous(), "bwd_gather_row", True)
            k_g, w4 = comm.col_all_gather(saved.k[:, sl].contiguous(), "bwd_gather_kv", True)
            v_g, w5 = comm.col_all_gather(saved.v[:, sl].contiguous(), "bwd_gather_kv", True)
            return (q_g, do_g, st_g, k_g, v_g), (w1, w2, w3, w4, w5)

        dq_parts, dk_parts, dv_parts = [], [], []
        reduce_work = []
        nxt = gathers(0)
        for i in range(len(chunks)):
            cur = nxt
            if i + 1 < len(chunks):
                nxt = gathers(i + 1)
            wait_all(cur[1])
            q_g, do_g, st_g, k_g, v_g = cur[0]
            bh = q_g.shape[1]
            lse_g = st_g[..., 0].t().contiguous()
            delta_g = st_g[..., 1].t().contiguous()
            dq_acc = torch.zeros((g.pc * L, bh, h), dtype=torch.float32, device=q_g.device)
            kdt = torch.float32 if g.pr > 1 else saved.q.dtype
            dk_g = torch.empty((g.pr * L, bh, h), dtype=kdt, device=q_g.device)
            dv_g = torch.empty((g.pr * L, bh, h), dtype=kdt, device=q_g.device)
            self.ops.tile_backward(_heads(q_g), _heads(k_g), _heads(v_g), _heads(do_g), lse_g,
                                   delta_g, causal=self.causal, scale=self.scale,
                                   q_index=self.q_index, k_index=self.k_index,
                                   dq_acc=_heads(dq_acc), dk=_heads(dk_g), dv=_heads(dv_g))
            dq, w1 = comm.row_reduce_scatter(dq_acc, async_op=True)
            dk, w2 = comm.col_reduce_scatter(dk_g, async_op=True)
            dv, w3 = comm.col_reduce_scatter(dv_g, async_op=True)
            dq_parts.append(dq)
            dk_parts.append(dk)
            dv_parts.append(dv)
            reduce_work.append((w1, w2, w3))
        wait_all(reduce_work)
        dq_acc = dq_parts[0] if len(chunks) == 1 else torch.cat(dq_parts, dim=1)
        dk_t = dk_parts[0] if len(chunks) == 1 else torch.cat(dk_parts, dim=1)
        dv_t = dv_parts[0] if len(chunks) == 1 else torch.cat(dv_parts, dim=1)
        dk_p, dv_p = comm.unpermute_kv(dk_t, dv_t)
        dt = saved.q.dtype
        dq_p = torch.empty((L, bh_all, h), dtype=dt, device=do_p.device)
        self.ops.bwd_finalize(_heads(dq_acc), self.scale, out=_heads(dq_p))
        return dq_p, dk_p.to(dt), dv_p.to(dt)


class _Attention2DFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q_p, k_p, v_p, plan: Attention2D):
        o_p, saved = plan.forward(q_p, k_p, v_p)
        ctx.plan = plan
        ctx.saved = saved
        return o_p

    @staticmethod
    def backward(ctx, do_p):
        dq, dk, dv = ctx.plan.backward(ctx.saved, do_p.to(ctx.saved.q.dtype).contiguous())
        return dq, dk, dv, None


def attention2d(q_p, k_p, v_p, plan: Attention2D) -> torch.Tensor:
    """Autograd entry point: rank-local shards [L, BH, H] in column-major
    cyclic layout (layouts.py) -> this rank's output rows."""
    return _Attention2DFn.apply(q_p, k_p, v_p, plan)
