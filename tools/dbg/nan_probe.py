import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2503_15758_b200 import ops
rng = np.random.default_rng(5)
q_idx = np.sort(rng.choice(600, size=150, replace=False))
k_idx = np.sort(rng.choice(np.arange(20, 600), size=260, replace=False))
for h in (64, 128):
    for causal in (True, False):
        for mode in ("array", "contig"):
            g = torch.Generator().manual_seed(30)
            q, k, v = ((torch.rand((2, n, h), generator=g) * 2 - 1).to(torch.bfloat16).cuda() for n in (150, 260, 260))
            if mode == "array":
                qi, ki = ops.TokenIndex.from_indices(q_idx), ops.TokenIndex.from_indices(k_idx)
            else:
                qi, ki = ops.TokenIndex.contiguous(150, 300), ops.TokenIndex.contiguous(260)
            for pm in (0, 1, 2):
                ops.debug_poison(pm)
                o, lse = ops.tile_forward(q, k, v, causal=causal, scale=0.125, q_index=qi, k_index=ki)
                torch.cuda.synchronize()
                bad = torch.isnan(o).any(-1)
                print(h, causal, mode, "poison", pm, "nan rows:", bad.sum().item(), torch.nonzero(bad)[:6].tolist(),
                      "lse nan", torch.isnan(lse).sum().item(), flush=True)
