import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2503_15758_b200 import ops
from gpu_util import uniform, ref_attention
rng = np.random.default_rng(11)
nq, nk = 300, 420
q_idx = np.sort(rng.choice(1000, size=nq, replace=False))
k_idx = np.sort(rng.choice(np.arange(30, 1000), size=nk, replace=False))
for h in (64, 128):
  for arr in (True, False):
    if arr:
        qi, ki = ops.TokenIndex.from_indices(q_idx), ops.TokenIndex.from_indices(k_idx)
        qg, kg = torch.from_numpy(q_idx), torch.from_numpy(k_idx)
    else:
        qi, ki = ops.TokenIndex.contiguous(nq, 500), ops.TokenIndex.contiguous(nk, 100)
        qg, kg = torch.arange(nq) + 500, torch.arange(nk) + 100
    q = uniform((2, nq, h), 70); k, v = uniform((2, nk, h), 72), uniform((2, nk, h), 73)
    want_o, want_lse = ref_attention(q, k, v, True, 0.1, qg, kg)
    for poison in (0, 1, 2, 3):
        o = torch.full((2, nq, h), float("nan"), device="cuda")
        lse = torch.full((2, nq), float("nan"), device="cuda")
        ops.debug_poison(poison)
        ops.tile_forward(q, k, v, causal=True, scale=0.1, q_index=qi, k_index=ki, out=o, lse=lse)
        torch.cuda.synchronize()
        err = (o - want_o.nan_to_num()).abs().amax(-1)
        bad = ~(err < 1e-2)
        rows = torch.nonzero(bad).tolist()
        print(h, "array" if arr else "affine", "poison", poison, "bad rows", len(rows), rows[:10],
              "lse bad", (~((lse - want_lse).abs() < 1e-3) & torch.isfinite(want_lse)).sum().item(), flush=True)
