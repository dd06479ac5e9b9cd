"""Producer-side cyclic layout: a layer whose per-token
producer (embedding + QKV projection) and consumer (output projection +
per-token loss) run on the data loader's cyclic shards feeds attention2d
directly — no relayout collective — and reproduces the single-device layer
on the contiguous sequence (loss and weight gradients), with the ledger
showing attention traffic only.  gloo ranks, CPU stand-in kernels."""

import os
import socket
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

N, D, M, H, VOCAB = 64, 32, 2, 16, 50


def _params():
    g = torch.Generator().manual_seed(0)
    emb = torch.randn(VOCAB, D, generator=g) * 0.5
    wqkv = torch.randn(D, 3 * M * H, generator=g) / D ** 0.5
    wo = torch.randn(M * H, D, generator=g) / (M * H) ** 0.5
    tokens = torch.randint(0, VOCAB, (N,), generator=g)
    return emb, wqkv, wo, tokens


def _layer(emb, wqkv, wo, tok, attend):
    x = emb[tok]                                   # per-token producer
    qkv = (x @ wqkv).view(-1, 3, M, H).to(torch.bfloat16)
    o = attend(qkv[:, 0].contiguous(), qkv[:, 1].contiguous(), qkv[:, 2].contiguous())
    y = o.float().reshape(-1, M * H) @ wo          # per-token consumer
    return (y * y).sum()


def _worker(rank, world, port, grid, outdir):
    sys.path.insert(0, str(HERE))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import cpu_compute
        from paper_2503_15758_b200.layouts import Grid2D
        from paper_2503_15758_b200.strategies import Attention2D, GridComm, attention2d
        from paper_2503_15758_b200.strategies.relayout import shard_tokens
        comm = GridComm(Grid2D(*grid))
        plan = Attention2D(comm, N, True, H ** -0.5, compute=cpu_compute)
        emb, wqkv, wo, tokens = (t.requires_grad_(t.is_floating_point()) for t in _params())
        tok = shard_tokens(tokens, comm)           # the loader's cyclic share
        loss = _layer(emb, wqkv, wo, tok, lambda q, k, v: attention2d(q, k, v, plan))
        loss.backward()
        tot = loss.detach().clone()
        dist.all_reduce(tot)
        grads = [t.grad.clone() for t in (emb, wqkv, wo)]
        for gr in grads:
            dist.all_reduce(gr)
        ops = sorted({op for (_, op) in comm.ledger.rows})
        if rank == 0:
            np.savez(Path(outdir) / "out.npz", loss=tot.numpy(), g0=grads[0].numpy(),
                     g1=grads[1].numpy(), g2=grads[2].numpy(), ops=np.array(ops))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("grid", [(2, 2), (1, 2), (2, 1)])
def test_cyclic_producer_layer_matches_single_device(grid):
    world = grid[0] * grid[1]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, port, grid, d), nprocs=world, join=True)
        got = dict(np.load(Path(d) / "out.npz"))
    # single device, contiguous sequence, dense causal attention in fp64
    sys.path.insert(0, str(HERE))
    emb, wqkv, wo, tokens = (t.requires_grad_(t.is_floating_point()) for t in _params())

    def dense(q, k, v):
        qf, kf, vf = (t.double().transpose(0, 1) for t in (q, k, v))   # [M, N, H]
        s = qf @ kf.transpose(1, 2) * H ** -0.5
        s = s.masked_fill(torch.ones(N, N, dtype=torch.bool).triu(1), float("-inf"))
        return (torch.softmax(s, -1) @ vf).transpose(0, 1)
    loss = _layer(emb, wqkv, wo, tokens, dense)
    loss.backward()
    ref = float(loss.detach())
    assert abs(float(got["loss"]) - ref) / abs(ref) < 2e-2
    for key, t in (("g0", emb), ("g1", wqkv), ("g2", wo)):
        want = t.grad.numpy()
        rel = np.linalg.norm(got[key] - want) / np.linalg.norm(want)
        assert rel < 3e-2, (key, rel)
    # no relayout collective at the layer boundary: attention traffic only
    assert not any(op in ("to_cyclic", "from_cyclic") for op in got["ops"])
