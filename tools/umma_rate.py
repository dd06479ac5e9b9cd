"""Measure tcgen05.mma issue rate per operand shape (diagnostic)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_15758_b200 import _lib  # noqa: E402
lib = _lib.load()
names = {0: "M128 N128 K/K", 1: "M128 N128 K/MN", 2: "M128 N64 K/K", 3: "M128 N64 MN/MN",
         4: "M128 N256 K/K", 5: "M128 N128 MN/MN", 6: "M128 N64 K/MN", 7: "TS M128 N128 B:K",
         8: "TS M128 N128 B:MN", 9: "TS M128 N64 B:K", 10: "TS M128 N256 B:K"}
ns = {0: 128, 1: 128, 2: 64, 3: 64, 4: 256, 5: 128, 6: 64, 7: 128, 8: 128, 9: 64, 10: 256}
iters = 2000
for ctas in (1, 148):
    for v in names:
        out = torch.zeros(ctas, dtype=torch.int64, device="cuda")
        lib.a2d_bench_umma(v, 10, out.data_ptr(), ctas, torch.cuda.current_stream().cuda_stream)
        lib.a2d_bench_umma(v, iters, out.data_ptr(), ctas, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        cyc = out.float().mean().item() / iters
        flops = 2 * 128 * ns[v] * 128
        print(f"ctas={ctas:3d} {names[v]:18s} {cyc:8.1f} cyc/unit(K=128)  {flops / cyc:7.0f} flop/cyc/SM"
              f"  (ideal {128 * ns[v] * 8 / 256:.0f} cyc)")
