"""Distributed attention strategies with the reference's contract
(pkg/src/attn2d/strategies/__init__.py:21-46):

    run_forward(name, cfg, q, k, v)      -> StrategyForward
    run_backward(name, cfg, saved, dout) -> StrategyBackward

Called collectively by every rank of the default process group (one rank
per GPU; a single process runs the 1-rank grid without torch.distributed).
Inputs and returned tensors are full (n, h) or (n, heads, h) arrays in
global token order, as in the reference; each rank computes only its shard
and the outputs are all-gathered back.  The rank-local entry points used by
training code and the benchmark are `Attention2D` / `attention2d` and
`Attention2DO` and `RingAttention`.

Strategies: "attn2d_no" (attn2d_no.py: collective gathers, head-chunk
pipelined), "attn2d_o" (attn2d_o.py: block rings overlapped with the tile
kernels, at most two live receive buffers per stream) and "ring" (the
same-kernel Ring Attention baseline).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from ..attention import count_unmasked
from ..errors import ConfigError
from ..layouts import Grid2D, ring_block_indices
from .attn2d_no import Attention2D, Saved2D, attention2d
from .attn2d_o import Attention2DO
from .comm import GridComm
from .common import DistAttnConfig, StrategyBackward, StrategyForward, assemble_rows
from .relayout import cyclic_token_ids, from_cyclic, shard_tokens, to_cyclic, unshard_tokens
from .ring import RingAttention

STRATEGY_NAMES = ("ring", "attn2d_no", "attn2d_o")
_COMMS: dict = {}


def get_strategy(name: str):
    if name == "attn2d_no":
        return Attention2D
    if name == "attn2d_o":
        return Attention2DO
    if name == "ring":
        return RingAttention
    raise ConfigError(f"unknown strategy {name!r}; expected one of {', '.join(STRATEGY_NAMES)}")


def _comm(grid: Grid2D) -> GridComm:
    key = (grid.pr, grid.pc, dist.is_initialized())
    if key not in _COMMS:
        _COMMS[key] = GridComm(grid)
    c = _COMMS[key]
    c.ledger.rows.clear()
    c.buffer_peaks.clear()
    return c


def _device():
    # gloo moves host tensors (the CPU tests); NCCL / single process: the GPU
    if dist.is_initialized() and dist.get_backend() == "gloo":
        return torch.device("cpu")
    if torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _as3(a, dev):
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))
    if t.dim() == 2:
        t = t[:, None, :]
    return t.to(dev)


def _grid_for(name: str, cfg: DistAttnConfig) -> Grid2D:
    if name in ("attn2d_no", "attn2d_o"):
        return cfg.grid2d()
    if cfg.p > 1 and cfg.n % (2 * cfg.p):
        raise ConfigError(f"ring layout needs 2*p={2 * cfg.p} to divide n={cfg.n}")
    return Grid2D(1, cfg.p)


def _owned(name, grid: Grid2D, n: int, rank: int) -> np.ndarray:
    if name == "ring":
        return ring_block_indices(n, grid.p, rank)
    return grid.owned(n, *grid.coord(rank))


def _scores(name, grid: Grid2D, n: int, causal: bool) -> dict:
    out = {}
    for rank in range(grid.p):
        r, c = grid.coord(rank)
        if name == "ring":
            qi = ring_block_indices(n, grid.p, rank)
            out[(r, c)] = count_unmasked(qi, np.arange(n), causal)
        else:
            out[(r, c)] = count_unmasked(grid.q_gathered(n, r).host(),
                                         grid.k_gathered(n, c).host(), causal)
    return out


def _gather_full(name, grid, n, local: torch.Tensor) -> torch.Tensor:
    if grid.p == 1:
        return local.clone()
    parts = [torch.empty_like(local) for _ in range(grid.p)]
    dist.all_gather(parts, local.contiguous())
    return assemble_rows(n, [(_owned(name, grid, n, rk), parts[rk]) for rk in range(grid.p)], local)


def run_forward(name: str, cfg: DistAttnConfig, q, k, v, compute=None) -> StrategyForward:
    cls = get_strategy(name)
    grid = _grid_for(name, cfg)
    comm = _comm(grid)
    dev = _device()
    idx = torch.as_tensor(_owned(name, grid, cfg.n, comm.rank), device=dev)
    q_p, k_p, v_p = (_as3(x, dev)[idx].to(torch.bfloat16).contiguous() for x in (q, k, v))
    plan = (cls(comm, cfg.n, cfg.causal, cfg.scale, head_chunks=cfg.head_chunks, compute=compute)
            if cls in (Attention2D, Attention2DO)
            else cls(comm, cfg.n, cfg.causal, cfg.scale, compute=compute))
    o_p, saved = plan.forward(q_p, k_p, v_p)
    o = _gather_full(name, grid, cfg.n, o_p.float())
    lse = _gather_full(name, grid, cfg.n, saved.lse)
    squeeze = (np.ndim(q) if not isinstance(q, torch.Tensor) else q.dim()) == 2
    return StrategyForward(o=o[:, 0] if squeeze else o, saved={"plan": plan, "state": saved,
                                                               "squeeze": squeeze},
                           ledger=comm.ledger, score_elements=_scores(name, grid, cfg.n,
                                                                      cfg.causal),
                           lse=lse[:, 0] if squeeze else lse,
                           buffer_peaks=dict(comm.buffer_peaks))


def run_backward(name: str, cfg: DistAttnConfig, saved, d_out) -> StrategyBackward:
    plan = saved["plan"]
    plan.comm.buffer_peaks.clear()
    grid = plan.comm.grid if hasattr(plan.comm, "grid") else Grid2D(1, cfg.p)
    dev = saved["state"].q.device
    idx = torch.as_tensor(_owned(name, grid, cfg.n, plan.comm.rank), device=dev)
    do_p = _as3(d_out, dev)[idx].to(torch.bfloat16).contiguous()
    dq_p, dk_p, dv_p = plan.backward(saved["state"], do_p)
    full = [_gather_full(name, grid, cfg.n, t.float()) for t in (dq_p, dk_p, dv_p)]
    if saved["squeeze"]:
        full = [t[:, 0] for t in full]
    return StrategyBackward(dq=full[0], dk=full[1], dv=full[2], ledger=plan.comm.ledger,
                            score_elements=_scores(name, grid, cfg.n, cfg.causal),
                            buffer_peaks=dict(plan.comm.buffer_peaks))


__all__ = ["STRATEGY_NAMES", "Attention2D", "Attention2DO", "DistAttnConfig", "GridComm", "RingAttention",
           "Saved2D", "StrategyBackward", "StrategyForward", "attention2d", "get_strategy",
           "run_backward", "run_forward", "to_cyclic", "from_cyclic", "cyclic_token_ids",
           "shard_tokens", "unshard_tokens"]
