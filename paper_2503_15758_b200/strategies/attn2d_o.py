"""Attention2D, overlapped schedule (reference strategies/attn2d_o.py;
PAPER Algs. 4-6 forward, 8-11 backward) on a Pr x Pc grid of B200s.

Same words on the wire as the non-overlapped schedule (attn2d_no.py), but no
rank ever waits for a whole gathered tensor before computing: every transfer
is one block, posted before the tile kernel that does not need it, so NCCL
moves block b+1 over NVLink while the tensor cores work on block b.

Forward on rank (r, c), shards [L, BH, H] token-major (L = N/P):
  1. permute K/V to the row-major residue (the mirror transpose);
  2. column sweep (gthr_cmpt, attn2d_o.py:34-81): the column's K/V blocks
     ring upward one hop per step, landing directly in their slice of the
     gathered buffer K_g(c); each block is folded into the partial of the
     rank's OWN query slice with the tile kernel's accumulate mode (attn_fix
     in place, :69-72);
  3. row sweep (gthr_cmpt_sctr, :84-123): the row's foreign query blocks ring
     left; each is run against the whole K_g(c) and its partial (O fp32,
     LSE) rides one hop left behind it, merged on arrival with the 2-way
     LSE-merge kernel, so the partial received last is the rank's own query
     slice over every other column's keys;
  4. own partial + that partial -> O, LSE (LSE-merge with finalize, :151-152).
Backward (:156-393): K/V re-stream up the column while the own (Q, dO, LSE,
delta) slice accumulates dQ and per-block dK/dV into K_g-shaped fp32
buffers; (Q, dO, LSE, delta) bundles ring left (delta replaces O, as in
attn2d_no.py), their dQ partials riding one hop behind; the last bundle is
processed one key slice at a time while dK/dV slices ring-reduce up the
column, so each rank's reduced slice arrives as its compute ends
(cmpt_sctr_bwd, :248-311); then the inverse permutation.

Each stream keeps at most two receive buffers live (the reference's
buffer discipline, test_strategies.py:346-360), tracked by GridComm.
Rectangular grids work unchanged (column rings have Pr members, row rings
Pc); the reference requires a square grid (:127).
"""

from __future__ import annotations

import torch

from .. import ops as _ops
from ..ops import TokenIndex
from .attn2d_no import Saved2D, _heads
from .comm import GridComm, wait_all


class Attention2DO:
    def __init__(self, comm: GridComm, n: int, causal: bool, scale: float, compute=None,
                 head_chunks: int = 1):
        self.comm = comm
        self.grid = g = comm.grid
        self.n = n
        self.L = g.check_n(n)
        self.causal = bool(causal)
        self.scale = float(scale)
        self.ops = compute if compute is not None else _ops
        r, c = comm.r, comm.c
        self.up = g.rank((r - 1) % g.pr, c)
        self.down = g.rank((r + 1) % g.pr, c)
        self.left = g.rank(r, (c - 1) % g.pc)
        self.right = g.rank(r, (c + 1) % g.pc)
        self.q_own = self._qblock(c)
        self.k_index = g.k_gathered(n, c)

    def _qblock(self, cc: int) -> TokenIndex:
        """Global rows of grid row r's query block held by column cc."""
        g = self.grid
        return TokenIndex.blocked([g.residue(self.comm.r, cc)], g.p, self.L)

    def _kblock(self, rr: int) -> TokenIndex:
        """Global rows of column c's key block held by grid row rr."""
        g = self.grid
        return TokenIndex.blocked([g.kv_residue(rr, self.comm.c)], g.p, self.L)

    def _blk(self, t: torch.Tensor, rr: int) -> torch.Tensor:
        return t[rr * self.L:(rr + 1) * self.L]

    # ------------------------------------------------------------------ fwd
    def forward(self, q_p: torch.Tensor, k_p: torch.Tensor, v_p: torch.Tensor):
        comm, g, L = self.comm, self.grid, self.L
        comm.phase = "attention_fwd"
        r, c = comm.r, comm.c
        bh, h = q_p.shape[1], q_p.shape[2]
        dev = q_p.device
        k_t, v_t = comm.permute_kv(k_p, v_p)
        q_next = None
        if g.pc > 1:  # the first foreign query block travels during the column sweep
            comm.buf_open("q")
            q_next = comm.exchange([q_p], self.left, self.right, "forward_q", async_op=True)
        k_g = torch.empty((g.pr * L, bh, h), dtype=k_t.dtype, device=dev)
        v_g = torch.empty_like(k_g)
        self._blk(k_g, r).copy_(k_t)
        self._blk(v_g, r).copy_(v_t)
        # fin[0]: own query slice over this column's keys; fin[1]: over the others
        fin_o = torch.empty((2, bh, L, h), dtype=torch.float32, device=dev)
        fin_l = torch.empty((2, bh, L), dtype=torch.float32, device=dev)
        for i in range(g.pr):
            rr = (r + i) % g.pr
            work = None
            if i < g.pr - 1:
                nr = (r + i + 1) % g.pr
                comm.buf_open("kv")
                _, work = comm.exchange([self._blk(k_g, rr), self._blk(v_g, rr)], self.up,
                                        self.down, "gather_kv", async_op=True,
                                        recv_into=[self._blk(k_g, nr), self._blk(v_g, nr)])
            self.ops.tile_forward(_heads(q_p), _heads(self._blk(k_g, rr)),
                                  _heads(self._blk(v_g, rr)), causal=self.causal,
                                  scale=self.scale, q_index=self.q_own,
                                  k_index=self._kblock(rr), out=fin_o[0], lse=fin_l[0],
                                  accumulate=i > 0)
            if i > 0:
                comm.buf_close("kv")  # block rr is folded (it stays in K_g for the row sweep)
            wait_all(work)
        if g.pc > 1:
            self._row_sweep_fwd(q_next, k_g, v_g, fin_o, fin_l)
            o_hm, lse_hm = self.ops.lse_merge(fin_o.view(2, bh * L, h), fin_l.view(2, bh * L),
                                              out_dtype=q_p.dtype)
        else:
            o_hm, lse_hm = self.ops.lse_merge(fin_o[:1].view(1, bh * L, h),
                                              fin_l[:1].view(1, bh * L), out_dtype=q_p.dtype)
        o_p = o_hm.view(bh, L, h).transpose(0, 1).contiguous()
        lse_p = lse_hm.view(bh, L).t().contiguous()
        return o_p, Saved2D(q=q_p, k=k_t, v=v_t, o=o_p, lse=lse_p)

    def _row_sweep_fwd(self, q_next, k_g, v_g, fin_o, fin_l):
        comm, g, L = self.comm, self.grid, self.L
        c = comm.c
        _, bh, L_, h = fin_o.shape
        dev = fin_o.device
        (cur_q,), qw = q_next
        wait_all(qw)
        pair_o = torch.empty((2, bh, L, h), dtype=torch.float32, device=dev)
        pair_l = torch.empty((2, bh, L), dtype=torch.float32, device=dev)
        scat = None
        for i in range(1, g.pc):
            cc = (c + i) % g.pc
            nxt = None
            if i < g.pc - 1:
                comm.buf_open("q")
                nxt = comm.exchange([cur_q], self.left, self.right, "forward_q", async_op=True)
            self.ops.tile_forward(_heads(cur_q), _heads(k_g), _heads(v_g), causal=self.causal,
                                  scale=self.scale, q_index=self._qblock(cc),
                                  k_index=self.k_index, out=pair_o[0], lse=pair_l[0])
            if scat is not None:  # fold the partial of block cc from the right (one hop behind)
                wait_all(scat)
                comm.buf_close("partial")
                mo, ml = self.ops.lse_merge(pair_o.view(2, bh * L, h), pair_l.view(2, bh * L),
                                            out_dtype=torch.float32)
                send_o, send_l = mo.view(bh, L, h), ml.view(bh, L)
            else:
                send_o, send_l = pair_o[0], pair_l[0]
            last = i == g.pc - 1
            nxt_pair = (torch.empty_like(pair_o), torch.empty_like(pair_l)) if not last else None
            into = [fin_o[1], fin_l[1]] if last else [nxt_pair[0][1], nxt_pair[1][1]]
            comm.buf_open("partial")
            _, scat = comm.exchange([send_o, send_l], self.left, self.right, "scatter_partial",
                                    async_op=True, recv_into=into)
            comm.buf_close("q")
            if nxt is not None:
                (cur_q,), qw = nxt
                wait_all(qw)
            if not last:
                pair_o, pair_l = nxt_pair
        wait_all(scat)
        comm.buf_close("partial")

    # ------------------------------------------------------------------ bwd
    def backward(self, saved: Saved2D, do_p: torch.Tensor):
        comm, g, L = self.comm, self.grid, self.L
        comm.phase = "attention_bwd"
        r, c = comm.r, comm.c
        bh, h = do_p.shape[1], do_p.shape[2]
        dev = do_p.device
        delta = self.ops.bwd_preprocess(_heads(saved.o), _heads(do_p))     # [BH, L]
        lse_hm = saved.lse.t().contiguous()                                 # [BH, L]
        stats = torch.stack([saved.lse, delta.t()], dim=-1).contiguous()   # [L, BH, 2]
        bundle_next = None
        if g.pc > 1:
            comm.buf_open("qod")
            bundle_next = comm.exchange([saved.q, do_p, stats], self.left, self.right,
                                        "forward_qod", async_op=True)
        k_g = torch.empty((g.pr * L, bh, h), dtype=saved.k.dtype, device=dev)
        v_g = torch.empty_like(k_g)
        self._blk(k_g, r).copy_(saved.k)
        self._blk(v_g, r).copy_(saved.v)
        dk_g = torch.empty((g.pr * L, bh, h), dtype=torch.float32, device=dev)
        dv_g = torch.empty_like(dk_g)
        dq_acc = torch.zeros((L, bh, h), dtype=torch.float32, device=dev)
        # column sweep (gthr_cmpt_bwd, :156-203)
        for i in range(g.pr):
            rr = (r + i) % g.pr
            work = None
            if i < g.pr - 1:
                nr = (r + i + 1) % g.pr
                comm.buf_open("kv")
                _, work = comm.exchange([self._blk(k_g, rr), self._blk(v_g, rr)], self.up,
                                        self.down, "gather_kv", async_op=True,
                                        recv_into=[self._blk(k_g, nr), self._blk(v_g, nr)])
            self.ops.tile_backward(_heads(saved.q), _heads(self._blk(k_g, rr)),
                                   _heads(self._blk(v_g, rr)), _heads(do_p), lse_hm, delta,
                                   causal=self.causal, scale=self.scale, q_index=self.q_own,
                                   k_index=self._kblock(rr), dq_acc=_heads(dq_acc),
                                   dk=_heads(self._blk(dk_g, rr)),
                                   dv=_heads(self._blk(dv_g, rr)))
            if i > 0:
                comm.buf_close("kv")
            wait_all(work)
        if g.pc > 1:
            dq2, dk_t, dv_t = self._row_sweep_bwd(bundle_next, k_g, v_g, dk_g, dv_g)
            dq_acc.add_(dq2)
        elif g.pr > 1:  # Pr x 1: no row sweep to hide the column reduction behind
            dk_t = comm.col_reduce_scatter(dk_g, "scatter_dkv")
            dv_t = comm.col_reduce_scatter(dv_g, "scatter_dkv")
        else:
            dk_t, dv_t = dk_g, dv_g
        dk_p, dv_p = comm.unpermute_kv(dk_t, dv_t)
        dt = saved.q.dtype
        dq_p = torch.empty((L, bh, h), dtype=dt, device=dev)
        self.ops.bwd_finalize(_heads(dq_acc), self.scale, out=_heads(dq_p))
        return dq_p, dk_p.to(dt), dv_p.to(dt)

    def _bwd_tile(self, bundle, q_index, k, v, k_index, dq, dk, dv, accumulate=False):
        q_b, do_b, st_b = bundle
        self.ops.tile_backward(_heads(q_b), _heads(k), _heads(v), _heads(do_b),
                               st_b[..., 0].t().contiguous(), st_b[..., 1].t().contiguous(),
                               causal=self.causal, scale=self.scale, q_index=q_index,
                               k_index=k_index, dq_acc=_heads(dq), dk=_heads(dk), dv=_heads(dv),
                               accumulate_dkv=accumulate)

    def _row_sweep_bwd(self, bundle_next, k_g, v_g, dk_g, dv_g):
        """gthr_cmpt_sctr_bwd (:314-372) with cmpt_sctr_bwd (:248-311) for the
        last bundle."""
        comm, g, L = self.comm, self.grid, self.L
        r, c = comm.r, comm.c
        dev = k_g.device
        bh, h = k_g.shape[1], k_g.shape[2]
        bundle, bw = bundle_next
        wait_all(bw)
        dq_recv = torch.empty((L, bh, h), dtype=torch.float32, device=dev)
        scat = None
        dk_fin = dv_fin = None
        for i in range(1, g.pc):
            cc = (c + i) % g.pc
            nxt = None
            if i < g.pc - 1:
                comm.buf_open("qod")
                nxt = comm.exchange(list(bundle), self.left, self.right, "forward_qod",
                                    async_op=True)
            dq_i = torch.zeros((L, bh, h), dtype=torch.float32, device=dev)
            if i < g.pc - 1 or g.pr == 1:
                # dK/dV of the gathered keys accumulate in place (kernel accumulate mode)
                self._bwd_tile(bundle, self._qblock(cc), k_g, v_g, self.k_index, dq_i, dk_g,
                               dv_g, accumulate=True)
                if i == g.pc - 1:
                    dk_fin, dv_fin = dk_g, dv_g
            else:
                dk_fin, dv_fin = self._last_bundle(bundle, self._qblock(cc), k_g, v_g, dk_g,
                                                   dv_g, dq_i)
            if scat is not None:  # dQ partial of block cc from the right, one hop behind
                wait_all(scat)
                comm.buf_close("dq")
                dq_i.add_(dq_recv)
                dq_recv = torch.empty_like(dq_recv)
            comm.buf_open("dq")
            _, scat = comm.exchange([dq_i], self.left, self.right, "scatter_dq", async_op=True,
                                    recv_into=[dq_recv])
            comm.buf_close("qod")
            if nxt is not None:
                bundle, bw = nxt
                wait_all(bw)
        wait_all(scat)
        comm.buf_close("dq")
        return dq_recv, dk_fin, dv_fin

    def _last_bundle(self, bundle, q_index, k_g, v_g, dk_g, dv_g, dq_i):
        """The last bundle one key slice at a time while dK/dV slices ring-reduce
        up the column: slice (r + j) % Pr is finished at step j and sent up,
        the own slice r last (cmpt_sctr_bwd, :248-311)."""
        comm, g, L = self.comm, self.grid, self.L
        r = comm.r
        inc_k = inc_v = None
        scat = None
        for j in list(range(1, g.pr)) + [0]:
            s = (r + j) % g.pr
            # this bundle's contribution is added in place to slice s of the
            # column sweep's dK/dV (kernel accumulate mode)
            dk_s, dv_s = self._blk(dk_g, s), self._blk(dv_g, s)
            self._bwd_tile(bundle, q_index, self._blk(k_g, s), self._blk(v_g, s), self._kblock(s),
                           dq_i, dk_s, dv_s, accumulate=True)
            if scat is not None:
                wait_all(scat)
                comm.buf_close("dkv")
                dk_s.add_(inc_k)
                dv_s.add_(inc_v)
            if j == 0:
                return dk_s, dv_s
            comm.buf_open("dkv")
            nk, nv = torch.empty_like(dk_s), torch.empty_like(dv_s)
            _, scat = comm.exchange([dk_s, dv_s], self.up, self.down, "scatter_dkv",
                                    async_op=True, recv_into=[nk, nv])
            inc_k, inc_v = nk, nv
        raise AssertionError("unreachable")
