import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2503_15758_b200 import ops
from gpu_util import uniform, ref_attention
rng = np.random.default_rng(11)
nq, nk, h = 300, 420, 128
q_idx = np.sort(rng.choice(1000, size=nq, replace=False))
k_idx = np.sort(rng.choice(np.arange(30, 1000), size=nk, replace=False))
qi, ki = ops.TokenIndex.from_indices(q_idx), ops.TokenIndex.from_indices(k_idx)
qg, kg = torch.from_numpy(q_idx), torch.from_numpy(k_idx)
q = uniform((2, nq, h), 70); k, v = uniform((2, nk, h), 72), uniform((2, nk, h), 73)
want_o, want_lse = ref_attention(q, k, v, True, 0.1, qg, kg)
o, lse = ops.tile_forward(q, k, v, causal=True, scale=0.1, q_index=qi, k_index=ki)
torch.cuda.synchronize()
print("q_idx[256:300]", q_idx[256:300].tolist())
print("k tile first idx", [int(k_idx[t*128]) for t in range(4)], "last", int(k_idx[-1]))
for r in (256, 260, 280, 299):
    a, b = o[0, r].double(), want_o[0, r].double().cuda()
    c = (a @ b / (b @ b)).item()
    print(r, "fit c", c, "resid", ((a - c * b).norm() / a.norm()).item(), "norms", a.norm().item(), b.norm().item())
    for t in range(4):
        sl = slice(t*128, min((t+1)*128, nk))
        kk = k[0, sl].double().cuda(); vv = v[0, sl].double().cuda()
        s = (q[0, r].double().cuda() @ kk.T) * 0.1
        s[torch.from_numpy(k_idx[sl] > q_idx[r]).cuda()] = -float("inf")
        w = torch.exp(s - want_lse[0, r].double().cuda())
        part = w @ vv
        e = a - b
        print("   tile", t, "contrib norm", part.norm().item(), "corr(err,part)", ((e @ part) / (part.norm() * e.norm() + 1e-30)).item(), "err norm", e.norm().item())
