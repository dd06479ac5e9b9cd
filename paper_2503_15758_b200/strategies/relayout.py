"""Token layout at the layer boundary (PAPER.md:376-380,
493-494, reference layouts.py:1-14).

Producer-side layout (no communication): the paper's data loader deals
tokens cyclically, so every per-token producer — embedding, QKV projection,
MLP, norms — already emits the column-major cyclic shard Attention2D reads,
and every per-token consumer takes its output as is.  `cyclic_token_ids`
gives the global token ids (= positions, e.g. for rotary embeddings) a rank
must load; `shard_tokens` / `unshard_tokens` are the loader-side gather and
the inverse used where a full sequence is assembled (host side, no device
traffic).  tests/test_layer_layout.py runs embedding -> QKV -> attention2d ->
output projection -> loss on cyclic shards and matches the single-device
contiguous layer with no relayout traffic in the ledger.

Relayout (one all_to_all each way), for stacks whose other layers insist on
contiguous sequence-parallel chunks:

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

import numpy as np
import torch
import torch.distributed as dist

from .comm import GridComm


def cyclic_token_ids(n: int, comm: GridComm, rank: int | None = None) -> np.ndarray:
    """Global token ids of rank's column-major cyclic shard, increasing:
    {x + P i} with x = residue(r, c) (layouts.py:53-65 generalised to Pr x Pc)."""
    g = comm.grid
    rk = comm.rank if rank is None else rank
    return g.owned(n, *g.coord(rk))


def shard_tokens(tokens, comm: GridComm):
    """The data loader's share of a sequence [N, ...] for this rank, already
    in the order Attention2D consumes (no relayout downstream)."""
    ids = cyclic_token_ids(tokens.shape[0], comm)
    return tokens[torch.as_tensor(ids)] if isinstance(tokens, torch.Tensor) else tokens[ids]


def unshard_tokens(parts: list, n: int, comm: GridComm):
    """Inverse of shard_tokens for per-rank results gathered on one host:
    parts[rank] -> full [N, ...] in sequence order."""
    out = torch.empty((n,) + tuple(parts[0].shape[1:]), dtype=parts[0].dtype)
    for rk, part in enumerate(parts):
        out[torch.as_tensor(cyclic_token_ids(n, comm, rk))] = part
    return out


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
