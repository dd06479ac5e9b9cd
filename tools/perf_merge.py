"""LSE-merge kernel timing at the 2x4 metric point: k_parts = Pc = 4
partials of rows = M * N/P per GPU (M=32, N=128K, P=8 -> 524288 rows), H=128.
Bytes per call = k*rows*(4H+4) read + rows*(2H+4) write.
usage: python tools/perf_merge.py [k_parts] [rows] [H]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_15758_b200 import ops  # noqa: E402


def main():
    kp = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    rows = int(sys.argv[2]) if len(sys.argv) > 2 else 32 * (131072 // 8)
    h = int(sys.argv[3]) if len(sys.argv) > 3 else 128
    o = torch.randn((kp, rows, h), device="cuda")
    lse = torch.randn((kp, rows), device="cuda")
    out = torch.empty((rows, h), dtype=torch.bfloat16, device="cuda")
    lo = torch.empty((rows,), device="cuda")
    for _ in range(3):
        ops.lse_merge(o, lse, out=out, lse_out=lo)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 20
    s.record()
    for _ in range(it):
        ops.lse_merge(o, lse, out=out, lse_out=lo)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / it
    nbytes = kp * rows * (4 * h + 4) + rows * (2 * h + 4)
    print(f"lse_merge k={kp} rows={rows} H={h}: {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s "
          f"(L2-resident partials? {kp * rows * 4 * h / 2**20:.0f} MiB read)")


if __name__ == "__main__":
    main()
