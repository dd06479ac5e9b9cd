import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2503_15758_b200 import ops
from gpu_util import uniform, ref_attention
h = 128
def run(q_idx, k_idx, tag, force_array=True):
    nq, nk = len(q_idx), len(k_idx)
    qi, ki = ops.TokenIndex.from_indices(q_idx), ops.TokenIndex.from_indices(k_idx)
    if force_array:
        qi, ki = qi.as_array("cuda"), ki.as_array("cuda")
    q = uniform((1, nq, h), 70); k, v = uniform((1, nk, h), 72), uniform((1, nk, h), 73)
    want_o, _ = ref_attention(q, k, v, True, 0.1, torch.from_numpy(q_idx), torch.from_numpy(k_idx))
    o, lse = ops.tile_forward(q, k, v, causal=True, scale=0.1, q_index=qi, k_index=ki)
    torch.cuda.synchronize()
    err = (o - want_o.nan_to_num()).abs().amax(-1)[0]
    bad = ~(err < 1e-2)
    tiles = sorted(set((torch.nonzero(bad)[:, 0] // 128).tolist()))
    print(tag, "nq", nq, "nk", nk, "bad rows", bad.sum().item(), "bad q tiles", tiles, flush=True)
rng = np.random.default_rng(11)
for nk in (128, 200, 256, 300, 384, 420, 512):
    q_idx = np.arange(300) + 700
    k_idx = np.arange(nk) + 100
    run(q_idx, k_idx, "contig-as-array")
for nq in (128, 256, 300, 384):
    q_idx = np.arange(nq) * 2 + 100
    k_idx = np.arange(420) * 2 + 50
    run(q_idx, k_idx, "stride2-as-array")
    run(q_idx, k_idx, "stride2-affine", force_array=False)
q_idx = np.sort(rng.choice(1000, size=300, replace=False))
k_idx = np.sort(rng.choice(np.arange(30, 1000), size=420, replace=False))
run(q_idx, k_idx, "random")
run(q_idx, k_idx[:384], "random-k384")
run(q_idx[:256], k_idx, "random-q256")
