"""Timeline of one bwd CTA from a -DTX/-DTY trace build (diagnostic)."""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_15758_b200 import ops  # noqa: E402
from paper_2503_15758_b200 import _lib  # noqa: E402

N, BH, H = int(sys.argv[1]), int(sys.argv[2]), 128
causal = bool(int(sys.argv[3]))
q, k, v, do = (torch.empty((BH, N, H), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
               for _ in range(4))
o, lse = ops.tile_forward(q, k, v, causal=causal, scale=H ** -0.5, out_dtype=torch.bfloat16)
delta = ops.bwd_preprocess(o, do)
for _ in range(2):
    ops.tile_backward(q, k, v, do, lse, delta, causal=causal, scale=H ** -0.5)
torch.cuda.synchronize()
buf = np.zeros((24, 1024), dtype=np.int64)
lib = _lib.load()
lib.a2d_trace_dump(ctypes.c_void_p(buf.ctypes.data))
names = ["S:looptop", "S:preqfull", "M:dofull", "M:pready", "M:dsready", "M:qfull+1", "M:dqfree",
         "S:qfull", "S:sfull", "S:P_arrive", "S:dpfull", "S:dsfree", "S:DS_arrive", "D:dqfull",
         "D:dqfree_arr", "D:last_commit", "B:P_arrive", "B:DS_arrive", "B:sfull", "B:dpfull",
         "", "", "", ""]
t0 = buf[buf > 0].min()
n = int((buf[8] > 0).sum())
print("iterations", n)
for i in list(range(0, 6)) + list(range(n // 2, n // 2 + 6)):
    print(f"i={i:3d} " + " ".join(f"{names[e].split(':')[1][:9]:>9s}={(buf[e, i] - t0) if buf[e, i] else -1:8d}"
                                  for e in range(20)))
d = lambda a, b: np.diff(buf[a, 1:n]).mean()
print("mean period (S:sfull)", np.diff(buf[8, 2:n - 2]).mean())
for e in range(20):
    if (buf[e, :n] > 0).sum() > 4:
        print(f"{names[e]:16s} mean delta vs S:sfull(i): {np.mean(buf[e, 2:n-2] - buf[8, 2:n-2]):9.0f}")
