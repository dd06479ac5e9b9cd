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
    line = json.loads((ROOT / "profiles" / "r1_bench_1gpu.json").read_text().strip())
    for key in ("roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    r = line["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] < 1.2 and r["unit"] == "TFLOP/s"
    assert line["gpu_launches"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
