"""Layer-boundary relayout between sequence-parallel contiguous chunks and
the column-major cyclic shards Attention2D consumes (the
paper assumes the data loader already deals tokens cyclically,
PAPER.md:376-380, 493-494, reference layouts.py:1-14).

Rank r of a Pr x Pc grid holds contiguous rows [r L, (r+1) L) (L = N/P) of a
token-major tensor; its cyclic shard is {x_r + P i} with x_r = residue(r).
When P divides L, every contiguous chunk holds exactly L/P rows of every
residue, so one all_to_all_single with equal splits moves each row straight
to its owner, and the rows arrive in increasing global order (source ranks
in order, strided rows within each).  The inverse is the same exchange
backwards.  Per-token producers and consumers (QKV / output projections,
MLP) are order-agnostic, so these two calls are the whole boundary cost.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .comm import GridComm


def _check(comm: GridComm, rows: int):
    p = comm.grid.p
    if rows % p:
        raise ValueError(f"{rows} rows per rank are not divisible by p={p} "
                         "(the relayout needs N % P^2 == 0)")
    return p, rows // p


def to_cyclic(x: torch.Tensor, comm: GridComm) -> torch.Tensor:
    """Contiguous chunk [L, ...] of this rank -> its cyclic shard [L, ...]."""
    g = comm.grid
    p, k = _check(comm, x.shape[0])
    if p == 1:
        return x
    # send block for destination rank d: my rows with t = x_d (mod P)
    parts = x.reshape(k, p, *x.shape[1:])
    order = [g.residue(*g.coord(d)) for d in range(p)]
    send = torch.stack([parts[:, res] for res in order], dim=0).contiguous()
    recv = torch.empty_like(send)
    comm.ledger.charge(comm.phase, "to_cyclic", send.numel() // p * (p - 1) * send.element_size(),
                       send.numel() // p * (p - 1) * send.element_size(),
                       send.numel() // p * (p - 1), p - 1)
    dist.all_to_all_single(recv.view(p * k, -1), send.view(p * k, -1), group=comm.world)
    return recv.reshape(p * k, *x.shape[1:])          # sources in order = global order


def from_cyclic(y: torch.Tensor, comm: GridComm) -> torch.Tensor:
    """Cyclic shard [L, ...] of this rank -> its contiguous chunk [L, ...]."""
    g = comm.grid
    p, k = _check(comm, y.shape[0])
    if p == 1:
        return y
    send = y.reshape(p, k, *y.shape[1:]).contiguous()  # block s: my rows inside chunk s
    recv = torch.empty_like(send)
    comm.ledger.charge(comm.phase, "from_cyclic", send.numel() // p * (p - 1) * send.element_size(),
                       send.numel() // p * (p - 1) * send.element_size(),
                       send.numel() // p * (p - 1), p - 1)
    dist.all_to_all_single(recv.view(p * k, -1), send.view(p * k, -1), group=comm.world)
    # recv block d = chunk rows with residue order[d]; interleave back by residue
    order = [g.residue(*g.coord(d)) for d in range(p)]
    out = torch.empty((k, p) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
    for d, res in enumerate(order):
        out[:, res] = recv[d]
    return out.reshape(p * k, *y.shape[1:])
