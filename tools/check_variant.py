"""Numerics of the library A2D_LIB_PATH points at (an xlib2/ variant) against a
torch fp32 reference: python tools/check_variant.py [N BH H causal]."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from gpu_util import ref_attention, ref_attention_grad, rel_fro  # noqa: E402
from paper_2503_15758_b200 import functional  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
BH = int(sys.argv[2]) if len(sys.argv) > 2 else 4
H = int(sys.argv[3]) if len(sys.argv) > 3 else 128
for causal in (True, False):
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, do = (torch.empty((BH, N, H), device="cuda").uniform_(-1, 1, generator=g)
                   .to(torch.bfloat16) for _ in range(4))
    qr, kr, vr = (x.clone().requires_grad_(True) for x in (q, k, v))
    o = functional.attention(qr, kr, vr, causal=causal)
    o.backward(do)
    ro, _ = ref_attention(q, k, v, causal, H ** -0.5)
    gq, gk, gv = ref_attention_grad(q, k, v, do, causal, H ** -0.5)
    errs = {n: rel_fro(a.float(), b) for n, a, b in (("O", o, ro), ("dQ", qr.grad, gq),
                                                     ("dK", kr.grad, gk), ("dV", vr.grad, gv))}
    ok = all(e < 1e-2 for e in errs.values())
    print(f"causal={causal} N={N} BH={BH} H={H} " +
          " ".join(f"{n}={e:.2e}" for n, e in errs.items()) + (" OK" if ok else " FAIL"))
