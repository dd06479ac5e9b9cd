"""Library context numbers (not the reference arm): torch SDPA with its
cuDNN / flash backends on the same shapes as tools/perf_tile.py, CUDA-event
timed.   usage: python tools/perf_sdpa.py N BH H causal [backend...]"""
import os
import sys

import torch
from torch.nn.attention import SDPBackend, sdpa_kernel

BACKENDS = {"cudnn": SDPBackend.CUDNN_ATTENTION, "flash": SDPBackend.FLASH_ATTENTION,
            "efficient": SDPBackend.EFFICIENT_ATTENTION}


def timeit(fn, iters=5, warm=2):
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
    N, BH, H = (int(x) for x in sys.argv[1:4])
    causal = bool(int(sys.argv[4]))
    names = sys.argv[5:] or ["cudnn"]
    q, k, v, do = (torch.empty((1, BH, N, H), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
                   for _ in range(4))
    pairs = N * (N + 1) // 2 if causal else N * N
    ffwd = 4.0 * H * pairs * BH
    for name in names:
        try:
            with sdpa_kernel(BACKENDS[name]):
                qq, kk, vv = (x.clone().requires_grad_(True) for x in (q, k, v))
                ms_f = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(
                    q, k, v, is_causal=causal))
                o = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=causal)

                def bwd():
                    torch.autograd.grad(o, (qq, kk, vv), do, retain_graph=True)
                if os.environ.get("SDPA_FWD_ONLY"):
                    print(f"{name}: fwd {ms_f:.3f} ms {ffwd / ms_f / 1e9:.1f} TFLOP/s")
                    continue
                ms_b = timeit(bwd)
            print(f"{name}: fwd N={N} BH={BH} H={H} causal={causal}: {ms_f:.3f} ms "
                  f"{ffwd / ms_f / 1e9:.1f} TFLOP/s | bwd {ms_b:.3f} ms {2.5 * ffwd / ms_b / 1e9:.1f} TFLOP/s")
        except Exception as exc:  # backend unavailable for this shape / build
            print(f"{name}: unavailable ({type(exc).__name__}: {str(exc)[:160]})")


if __name__ == "__main__":
    main()
