"""GPU bridge for the multi-rank strategy tests on a one-GPU box.

The strategies run over gloo on CPU tensors (one process per rank); every
kernel call they make is executed by the CUDA extension
(paper_2503_15758_b200.ops) on cuda:0 with the exact shapes, strides, index
maps and accumulate flags the strategy passed, and the results are copied
back into the caller's tensors.  So the N>1 call patterns of attn2d_no,
attn2d_o and ring are checked on the real sm_100a kernels even though NCCL
cannot put several ranks on one GPU.  Test infrastructure only.
"""

from __future__ import annotations

import torch

from paper_2503_15758_b200 import ops

DEV = torch.device("cuda", 0)


def _g(t):
    if t is None:
        return None
    g = torch.empty_strided(t.size(), t.stride(), dtype=t.dtype, device=DEV)
    g.copy_(t)
    return g


def _back(dst, src):
    if dst is None:
        return src.cpu()
    dst.copy_(src)
    return dst


def tile_forward(q, k, v, *, causal, scale, q_index=None, k_index=None, out=None, lse=None,
                 out_dtype=torch.float32, accumulate=False):
    og, lg = ops.tile_forward(_g(q), _g(k), _g(v), causal=causal, scale=scale, q_index=q_index,
                              k_index=k_index, out=_g(out), lse=_g(lse), out_dtype=out_dtype,
                              accumulate=accumulate)
    torch.cuda.synchronize()
    return _back(out, og), _back(lse, lg)


def lse_merge(o_parts, lse_parts, *, out=None, lse_out=None, out_dtype=torch.bfloat16):
    og, lg = ops.lse_merge(_g(o_parts), _g(lse_parts), out_dtype=out_dtype)
    torch.cuda.synchronize()
    return _back(out, og), _back(lse_out, lg)


def bwd_preprocess(o, dout):
    d = ops.bwd_preprocess(_g(o), _g(dout))
    torch.cuda.synchronize()
    return d.cpu()


def tile_backward(q, k, v, dout, lse, delta, *, causal, scale, q_index=None, k_index=None,
                  dq_acc=None, dk=None, dv=None, dkv_dtype=torch.float32, accumulate_dkv=False):
    dqg, dkg, dvg = ops.tile_backward(_g(q), _g(k), _g(v), _g(dout), _g(lse), _g(delta),
                                      causal=causal, scale=scale, q_index=q_index,
                                      k_index=k_index, dq_acc=_g(dq_acc), dk=_g(dk), dv=_g(dv),
                                      dkv_dtype=dkv_dtype, accumulate_dkv=accumulate_dkv)
    torch.cuda.synchronize()
    return _back(dq_acc, dqg), _back(dk, dkg), _back(dv, dvg)


def bwd_finalize(dq_acc, scale, out=None, dtype=torch.bfloat16):
    og = ops.bwd_finalize(_g(dq_acc), scale, out=_g(out))
    torch.cuda.synchronize()
    return _back(out, og)
