"""Timeline of one fwd2 CTA from an A2D_TRACE build (diagnostic).
usage: A2D_LIB_PATH=xlib2/lib_ftrace.so python tools/trace_fwd2.py N BH causal
(build: python tools/mk_variant.py ftrace)"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_15758_b200 import ops  # noqa: E402
from paper_2503_15758_b200 import _lib  # noqa: E402

N, BH, H = int(sys.argv[1]), int(sys.argv[2]), 128
causal = bool(int(sys.argv[3]))
q, k, v = (torch.empty((BH, N, H), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
           for _ in range(3))
for _ in range(3):
    ops.tile_forward(q, k, v, causal=causal, scale=H ** -0.5, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
buf = np.zeros((48, 1024), dtype=np.int64)
lib = _lib.load()
lib.a2d_trace_dump(ctypes.c_void_p(buf.ctypes.data))
n = int((buf[40] > 0).sum())
t0 = buf[buf > 0].min()
print("tiles", n)
ev = ["sfull", "ld", "max", "exp", "arrive"]
def row(e, t, qq):
    return buf[e * 8 + t * 4 + qq, :n]
for j in list(range(0, 4)) + list(range(n // 2, n // 2 + 4)):
    line = f"j={j:3d} "
    for t in range(2):
        line += f"| T{t} " + " ".join(f"{ev[e]}={row(e, t, 0)[j] - t0:7d}" for e in range(5))
        line += f" arr[q0..3]=" + ",".join(str(row(4, t, qq)[j] - t0) for qq in range(4))
    line += f" | M: vfull={buf[44, j] - t0} p0={buf[40, j] - t0} qk0={buf[41, j] - t0} p1={buf[42, j] - t0} qk1={buf[43, j] - t0}"
    print(line)
m = slice(2, n - 2)
print("period (T0 sfull)", np.diff(buf[0, 2:n - 2]).mean())
for t in range(2):
    for qq in range(4):
        s = row(0, t, qq)
        print(f"T{t} warp{qq}: ld {np.mean(row(1,t,qq)[m]-s[m]):6.0f} max {np.mean(row(2,t,qq)[m]-s[m]):6.0f} "
              f"exp {np.mean(row(3,t,qq)[m]-s[m]):6.0f} arrive {np.mean(row(4,t,qq)[m]-s[m]):6.0f}")
arr0 = np.max([row(4, 0, qq) for qq in range(4)], axis=0)
arr1 = np.max([row(4, 1, qq) for qq in range(4)], axis=0)
print("MMA wake after last P0 arrive", np.mean(buf[40, m] - arr0[m]))
print("MMA wake after last P1 arrive", np.mean(buf[42, m] - arr1[m]))
print("S0(j+1) sfull after qk0(j) issued", np.mean(buf[0, 3:n - 1] - buf[41, 2:n - 2]))
print("S1(j+1) sfull after qk1(j) issued", np.mean(buf[4, 3:n - 1] - buf[43, 2:n - 2]))
print("qk0 issue - p0 wake", np.mean(buf[41, m] - buf[40, m]), " qk1 issue - p1 wake", np.mean(buf[43, m] - buf[42, m]))
