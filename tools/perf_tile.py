"""Quick tile-kernel timing (CUDA events, warm-up, L2-sized inputs).
usage: python tools/perf_tile.py [fwd|bwd|all] N BH H causal"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_15758_b200 import ops  # noqa: E402


def timeit(fn, iters=int(__import__("os").environ.get("A2D_PERF_ITERS", "5")), warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "fwd"
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
    BH = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    H = int(sys.argv[4]) if len(sys.argv) > 4 else 128
    causal = bool(int(sys.argv[5])) if len(sys.argv) > 5 else True
    q, k, v, do = (torch.empty((BH, N, H), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
                   for _ in range(4))
    pairs = N * (N + 1) // 2 if causal else N * N
    ffwd = 4.0 * H * pairs * BH
    scale = H ** -0.5
    o = torch.empty_like(q)
    lse = torch.empty((BH, N), device="cuda")
    if what in ("fwd", "all"):
        ms = timeit(lambda: ops.tile_forward(q, k, v, causal=causal, scale=scale, out=o, lse=lse))
        print(f"fwd N={N} BH={BH} H={H} causal={causal}: {ms:.3f} ms  {ffwd / ms / 1e9:.1f} TFLOP/s")
    if what in ("bwd", "all"):
        ops.tile_forward(q, k, v, causal=causal, scale=scale, out=o, lse=lse)
        dq_acc = torch.zeros((BH, N, H), device="cuda")
        dk = torch.empty_like(q)
        dv = torch.empty_like(q)

        def bwd():
            delta = ops.bwd_preprocess(o, do)
            dq_acc.zero_()
            ops.tile_backward(q, k, v, do, lse, delta, causal=causal, scale=scale, dq_acc=dq_acc,
                              dk=dk, dv=dv)
            ops.bwd_finalize(dq_acc, scale)
        ms = timeit(bwd)
        print(f"bwd N={N} BH={BH} H={H} causal={causal}: {ms:.3f} ms  {2.5 * ffwd / ms / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
