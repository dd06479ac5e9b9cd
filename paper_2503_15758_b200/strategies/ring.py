"""Ring Attention baseline on the same tile kernel (reference
strategies/ring.py; PAPER §4, TE load-balanced layout).

Rank k keeps its query rows (front block k + mirrored back block,
ring.py:27-38) and the K/V blocks circulate P-1 hops.  Unlike the reference
(blocking send_recv after each fold, :77-79) the next hop is prefetched into
a second buffer while the current tile runs, so the baseline is a fair,
overlapped ring:
  forward: partials fold in place — the tile kernel's accumulate mode merges
           each hop into the running (O, LSE) state (attn_fix, :69-76);
  backward: (K, V) circulate ahead of compute; the (dK, dV) accumulator of a
           block travels with it one hop behind (:118-143), plus one home hop.
"""

from __future__ import annotations

import torch

from .. import ops as _ops
from ..layouts import ring_index
from .attn2d_no import Saved2D, _heads
from .comm import GridComm, wait_all


class RingAttention:
    def __init__(self, comm: GridComm, n: int, causal: bool, scale: float, compute=None):
        self.comm = comm
        self.p = comm.grid.p
        self.rank = comm.rank
        self.n = n
        self.causal = bool(causal)
        self.scale = float(scale)
        self.ops = compute if compute is not None else _ops
        self.nxt = (self.rank + 1) % self.p
        self.prv = (self.rank - 1) % self.p
        self.q_index = ring_index(n, self.p, self.rank)

    def forward(self, q_p, k_p, v_p):
        comm = self.comm
        comm.phase = "attention_fwd"
        rows, bh, h = q_p.shape
        o = torch.empty((rows, bh, h), dtype=torch.float32, device=q_p.device)
        lse = torch.empty((bh, rows), dtype=torch.float32, device=q_p.device)
        cur_k, cur_v, src = k_p, v_p, self.rank
        for step in range(self.p):
            work = None
            if step < self.p - 1:
                (nk, nv), work = comm.exchange([cur_k, cur_v], self.nxt, self.prv, "ring_kv", True)
            self.ops.tile_forward(_heads(q_p), _heads(cur_k), _heads(cur_v), causal=self.causal,
                                  scale=self.scale, q_index=self.q_index,
                                  k_index=ring_index(self.n, self.p, src), out=_heads(o), lse=lse,
                                  accumulate=step > 0)
            if work is not None:
                wait_all(work)
                cur_k, cur_v = nk, nv
            src = (src - 1) % self.p
        o_p = o.to(q_p.dtype)
        lse_p = lse.t().contiguous()
        return o_p, Saved2D(q=q_p, k=k_p, v=v_p, o=o_p, lse=lse_p)

    def backward(self, saved: Saved2D, do_p):
        comm = self.comm
        comm.phase = "attention_bwd"
        rows, bh, h = do_p.shape
        delta = self.ops.bwd_preprocess(_heads(saved.o), _heads(do_p))
        lse = saved.lse.t().contiguous()
        dq_acc = torch.zeros((rows, bh, h), dtype=torch.float32, device=do_p.device)
        dk_acc = torch.empty((rows, bh, h), dtype=torch.float32, device=do_p.device)
        dv_acc = torch.empty_like(dk_acc)
        dk_tmp = torch.empty_like(dk_acc)
        dv_tmp = torch.empty_like(dk_acc)
        cur_k, cur_v, src = saved.k, saved.v, self.rank
        acc_work = None
        for step in range(self.p):
            kv_work = None
            if step < self.p - 1:
                (nk, nv), kv_work = comm.exchange([cur_k, cur_v], self.nxt, self.prv, "ring_kv",
                                                  True)
            # Step 0 writes the own block's accumulator directly.  Later steps
            # write a scratch block and add it once the travelling accumulator
            # of block `src` has arrived: accumulating in place would make the
            # kernel wait for that hop (its sender finishes the previous step
            # at the same time as this rank), exposing the transfer.
            first = step == 0
            self.ops.tile_backward(_heads(saved.q), _heads(cur_k), _heads(cur_v), _heads(do_p),
                                   lse, delta, causal=self.causal, scale=self.scale,
                                   q_index=self.q_index, k_index=ring_index(self.n, self.p, src),
                                   dq_acc=_heads(dq_acc), dk=_heads(dk_acc if first else dk_tmp),
                                   dv=_heads(dv_acc if first else dv_tmp))
            if acc_work is not None:  # the accumulator of block `src` arrives from prev
                wait_all(acc_work[1])
                dk_acc, dv_acc = acc_work[0]
            if not first:
                dk_acc.add_(dk_tmp)
                dv_acc.add_(dv_tmp)
            if self.p > 1:
                # forward this block's accumulator (after P-1 hops it is one short of home)
                acc_work = comm.exchange([dk_acc, dv_acc], self.nxt, self.prv,
                                         "ring_kvg" if step < self.p - 1 else "ring_home", True)
            if kv_work is not None:
                wait_all(kv_work)
                cur_k, cur_v = nk, nv
            src = (src - 1) % self.p
        if acc_work is not None:
            wait_all(acc_work[1])
            dk_acc, dv_acc = acc_work[0]
        dt = saved.q.dtype
        dq_p = torch.empty((rows, bh, h), dtype=dt, device=do_p.device)
        self.ops.bwd_finalize(_heads(dq_acc), self.scale, out=_heads(dq_p))
        return dq_p, dk_acc.to(dt), dv_acc.to(dt)
