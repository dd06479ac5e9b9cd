"""bench.py driver contract, checked on CPU through the reference arm (the
oracle port of the reference's CPU kernels): one JSON line with the keys the
driver reads.  The GPU arm's line is produced on the B200 (profiles/)."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_prints_one_contract_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, check=True).stdout.strip().splitlines()
    assert len(out) == 1
    line = json.loads(out[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["unit"] == "TFLOP/s" and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] in ("port", "reference")
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_gpu_line_in_profiles_has_the_contract_keys():
    line = json.loads((ROOT / "profiles" / "r2_bench_1gpu.json").read_text().strip())
    for key in ("roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    r = line["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] < 1.2 and r["unit"] == "TFLOP/s"
    assert line["gpu_launches"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0


def _dist_worker(rank, world, port, outdir):
    import os
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import bench
        import cpu_compute
        args = bench.parse_args(["--gpus", str(world), "--seq-len", "256", "--heads", "2",
                                 "--head-dim", "16", "--steps", "2", "--warmup", "1",
                                 "--head-chunks", "2"])
        mark, elapsed = bench.cpu_marks()
        res = bench.run_dist(args, rank, world, torch.device("cpu"), cpu_compute, mark, elapsed,
                             lambda: None)
        fields = bench.dist_line_fields(args, res, world, torch.device("cpu"),
                                        bench.measured_peaks())
        if rank == 0:
            (Path(outdir) / "line.json").write_text(json.dumps(
                {k: v for k, v in fields.items() if k != "plan"}, default=str))
    finally:
        dist.destroy_process_group()


def test_multi_rank_path_on_gloo():
    """The N > 1 measurement path of bench.py (strategy arm + same-kernel
    Ring arm, per-rank kernel intervals -> roofline, byte / message ledger,
    max over ranks) with gloo and the CPU stand-in for the kernels."""
    import socket
    import tempfile

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_dist_worker, args=(2, port, d), nprocs=2, join=True)
        line = json.loads((Path(d) / "line.json").read_text())
    assert line["value"] > 0 and line["ms_per_step"] > 0
    r = line["roofline"]
    assert r["kernel"].startswith("tile_bwd") and r["achieved"] > 0 and len(r["per_rank_tflops"]) == 2
    # causal pairs of a 2x1 grid: each rank's bwd work is half the total
    total = 10.0 * 2 * 16 * (256 * 257 // 2)
    assert abs(r["flops_per_step_rank"] - total / 2) / total < 0.02
    assert line["comm"]["bytes_out_per_rank_per_step_max"] > 0
    assert line["comm"]["messages_per_rank_per_step_max"] > 0
    assert line["ring"]["value"] > 0 and line["vs_ring"] > 0


def test_gpus_flag_fails_loudly_without_devices():
    """--gpus N outside torchrun launches N ranks itself; with fewer CUDA
    devices than requested it must fail, not silently run 1 GPU."""
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode != 0 and "CUDA devices" in (p.stderr + p.stdout)
