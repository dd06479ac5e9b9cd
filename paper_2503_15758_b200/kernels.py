"""Drop-in for the reference's kernel module (pkg/src/attn2d/kernels/__init__.py).

Same function names, argument meaning and in-place output contract; one
implementation only (the sm_100a kernels) — there is no backend dispatch and
no CPU fallback.  `use_backend` accepts "auto" / "b200" and rejects anything
else with ValueError, like the reference does for unknown names
(kernels/__init__.py:37-46).

State conversion: the reference carries (m, nacc, d) per row; the kernels
carry (O, LSE).  flash_forward reads a live state as O = nacc / d,
LSE = m + log d, continues it on the device (accumulate mode), and writes
back the canonical triple (m, nacc, d) = (LSE, O, 1) — equal in every
observable (finalize, logsumexp, attn_fix) to the reference's.
"""

from __future__ import annotations

import numpy as np
import torch

from . import ops
from .attention import _padded_h, _to_bf16, _device

_NAME = "b200"


def use_backend(name: str) -> str:
    if name not in ("auto", _NAME):
        raise ValueError(f"unknown kernel backend {name!r}; have {[_NAME]}")
    return _NAME


def backend_name() -> str:
    return _NAME


def available_backends() -> tuple[str, ...]:
    return (_NAME,)


def _tensor(a) -> torch.Tensor:
    return a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))


def _write_back(dst, value: torch.Tensor) -> None:
    if isinstance(dst, torch.Tensor):
        dst.copy_(value.to(dst.device, dst.dtype))
    else:
        dst[...] = value.detach().cpu().numpy().astype(dst.dtype, copy=False)


def matmul(a, b, out) -> None:
    """out <- a @ b (dense-oracle helper of the reference; library GEMM)."""
    _write_back(out, _tensor(a).to(_device(), torch.float64) @ _tensor(b).to(_device(), torch.float64))


def matmul_t(a, b, out) -> None:
    """out <- a @ b.T."""
    _write_back(out, _tensor(a).to(_device(), torch.float64)
                @ _tensor(b).to(_device(), torch.float64).T)


def flash_forward(q, k, v, q_idx, k_idx, causal, scale, block, m, nacc, d) -> None:
    """Blockwise attention forward, updating (m, nacc, d) in place
    (kernels/__init__.py:70-78)."""
    dev = _device()
    qt, kt, vt = _tensor(q), _tensor(k), _tensor(v)
    nq, h = qt.shape
    hp = _padded_h(max(h, 1))
    mt = _tensor(m).to(dev, torch.float64)
    dt = _tensor(d).to(dev, torch.float64)
    nt = _tensor(nacc).to(dev, torch.float64)
    live = dt > 0
    state_o = torch.zeros((1, nq, hp), dtype=torch.float32, device=dev)
    state_o[0, :, :h] = torch.where(live[:, None], nt / torch.where(live, dt, 1.0)[:, None],
                                    0.0).to(torch.float32)
    state_lse = torch.where(live, mt + torch.log(torch.where(live, dt, 1.0)),
                            torch.full_like(mt, float("-inf"))).to(torch.float32)[None].contiguous()
    if kt.shape[0] > 0 and nq > 0:
        qi = ops.TokenIndex.from_indices(q_idx, dev)
        ki = ops.TokenIndex.from_indices(k_idx, dev)
        ops.tile_forward(_to_bf16(qt, hp), _to_bf16(kt, hp), _to_bf16(vt, hp), causal=bool(causal),
                         scale=float(scale), q_index=qi, k_index=ki, out=state_o, lse=state_lse,
                         accumulate=True)
    lse = state_lse[0].to(torch.float64)
    alive = torch.isfinite(lse)
    _write_back(m, lse)
    _write_back(d, alive.to(torch.float64))
    _write_back(nacc, state_o[0, :, :h].to(torch.float64) * alive[:, None])


def flash_backward(q, k, v, o, d_out, m_stat, d_stat, q_idx, k_idx, causal, scale, dq, dk, dv):
    """Accumulate gradients into dq/dk/dv from GLOBAL row statistics
    (kernels/__init__.py:81-92)."""
    dev = _device()
    qt, kt, vt = _tensor(q), _tensor(k), _tensor(v)
    h = qt.shape[1]
    hp = _padded_h(max(h, 1))
    lse = (_tensor(m_stat).to(dev, torch.float64) +
           torch.log(_tensor(d_stat).to(dev, torch.float64))).to(torch.float32)[None].contiguous()
    ob, dob = _to_bf16(_tensor(o), hp), _to_bf16(_tensor(d_out), hp)
    qi = ops.TokenIndex.from_indices(q_idx, dev)
    ki = ops.TokenIndex.from_indices(k_idx, dev)
    delta = ops.bwd_preprocess(ob, dob)
    dq_acc, dkk, dvv = ops.tile_backward(_to_bf16(qt, hp), _to_bf16(kt, hp), _to_bf16(vt, hp), dob,
                                         lse, delta, causal=bool(causal), scale=float(scale),
                                         q_index=qi, k_index=ki)
    for dst, val in ((dq, dq_acc[0, :, :h] * float(scale)), (dk, dkk[0, :, :h]), (dv, dvv[0, :, :h])):
        cur = _tensor(dst).to(dev, torch.float64)
        _write_back(dst, cur + val.to(torch.float64))
