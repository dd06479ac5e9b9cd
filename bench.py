"""Attention2D benchmark — the driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--strategy attn2d_no|attn2d_o|ring]

Workload (BASELINE.json metric): exact causal attention forward+backward at
N = 131072 tokens, M = 32 heads, H = 128, B = 1, bf16 — one step is one
fwd+bwd of that layer over the whole sequence, on an N-GPU Pr x Pc grid
(1 -> 1x1, 2 -> 2x1, 4 -> 2x2, 8 -> 2x4), synthetic uniform[-1, 1] inputs.
FLOPs follow BASELINE.md §3: 4·B·M·H·N(N+1)/2 forward, x3.5 forward+backward
(count_unmasked, attention.py:260-265).  Every input tensor is 1 GiB
(> 126 MB L2), so no L2 flush is needed between steps.

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GRIDS = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (2, 4)}
METRIC = "attention fwd+bwd TFLOP/s at N=128K on 1/2/4/8 B200; speedup vs Ring Attention"


def flops_fwd(b, m, h, n, causal=True):
    pairs = n * (n + 1) // 2 if causal else n * n
    return 4.0 * b * m * h * pairs


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), \
            d.get("hbm_gbs", 6650.0), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.lines: list[str] = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons, power = [], [], set(), []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------------------------
# CPU legs: the oracle port of the reference's numpy kernels
# --------------------------------------------------------------------------

def cpu_sample(n_cpu=4096, h=128, causal=True, budget_s=12.0, max_heads=32):
    """Time the reference algorithm (oracle port of kernels/numpy_backend.py,
    fwd + bwd through flash_attn_forward / finalize / flash_attn_backward) on
    a bounded sample: whole heads of N=n_cpu until the budget is spent."""
    import numpy as np
    from oracle import attn2d_oracle as orc

    rng = np.random.default_rng(0)
    idx = np.arange(n_cpu)
    heads, t0 = 0, time.perf_counter()
    while heads < max_heads and (heads == 0 or time.perf_counter() - t0 < budget_s):
        q, k, v, do = (rng.uniform(-1, 1, (n_cpu, h)) for _ in range(4))
        o, lse, (m, d) = orc.tile_forward_full(q, k, v, idx, idx, causal, h ** -0.5, block=64)
        orc.tile_backward_full(q, k, v, o, do, m, d, idx, idx, causal, h ** -0.5)
        heads += 1
    dt = time.perf_counter() - t0
    fl = 3.5 * flops_fwd(1, heads, h, n_cpu, causal)
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": os.cpu_count(),
            "kind": "port", "seconds": dt,
            "sample": f"{heads} head(s) of N={n_cpu}, H={h}, causal fwd+bwd, fp64 numpy "
                      f"(oracle port of kernels/numpy_backend.py), BLAS threads = all host cores"}


def run_reference(args, rank):
    """--impl reference: the reference's CPU algorithm on the host cores."""
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_sample(budget_s=0.0, max_heads=1)
    vals = []
    for _ in range(args.steps):
        s = cpu_sample(budget_s=0.0, max_heads=1)
        vals.append(s)
    v = statistics.median(x["value"] for x in vals)
    ms = statistics.median(x["seconds"] for x in vals) * 1e3
    cb = dict(vals[0])
    cb["value"] = v
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic uniform[-1,1]",
        "config": {"workload": "causal attention fwd+bwd, reference CPU algorithm, bounded "
                               "sample of the N=131072 M=32 H=128 layer (1 head of N=4096 "
                               "per step)", "seq_len_sample": 4096, "heads_sample": 1,
                   "head_dim": 128, "causal": True},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2503_15758_b200 import _lib, functional, ops
    from paper_2503_15758_b200.layouts import Grid2D
    from paper_2503_15758_b200.strategies import Attention2D, Attention2DO, GridComm, RingAttention

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    _lib.load()
    N, M, H, B = args.seq_len, args.heads, 128, 1
    BH = B * M
    causal = not args.non_causal
    scale = H ** -0.5
    pr, pc = GRIDS.get(world, (1, world))
    if args.grid:
        pr, pc = (int(x) for x in args.grid.lower().split("x"))
        if pr * pc != world:
            raise SystemExit(f"--grid {args.grid} does not match {world} ranks")
    grid = Grid2D(pr, pc) if args.strategy in ("attn2d_no", "attn2d_o") else Grid2D(1, world)
    L = N // world
    g = torch.Generator(device=dev).manual_seed(1234 + rank)

    def rnd(shape):
        return torch.empty(shape, dtype=torch.bfloat16, device=dev).uniform_(-1, 1, generator=g)

    fl_step = (1.0 if args.fwd_only else 3.5) * flops_fwd(B, M, H, N, causal)
    stream = torch.cuda.current_stream()

    # kernel-level events for the roofline of the dominant kernel (tile bwd)
    kev = {"bwd": [], "fwd": []}

    if world == 1:
        q, k, v, do = (rnd((BH, N, H)) for _ in range(4))
        dq_acc = torch.zeros((BH, N, H), dtype=torch.float32, device=dev)
        o = torch.empty_like(q)
        lse = torch.empty((BH, N), dtype=torch.float32, device=dev)
        dk, dv = torch.empty_like(k), torch.empty_like(v)
        dq = torch.empty_like(q)

        def step(record=False):
            e0 = torch.cuda.Event(enable_timing=True) if record else None
            if record:
                e0.record(stream)
            ops.tile_forward(q, k, v, causal=causal, scale=scale, out=o, lse=lse,
                             out_dtype=torch.bfloat16)
            if record:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
            if args.fwd_only:
                if record:
                    kev["fwd"].append((e0, e1))
                return
            delta = ops.bwd_preprocess(o, do)
            dq_acc.zero_()
            if record:
                e2 = torch.cuda.Event(enable_timing=True)
                e2.record(stream)
            ops.tile_backward(q, k, v, do, lse, delta, causal=causal, scale=scale, dq_acc=dq_acc,
                              dk=dk, dv=dv)
            if record:
                e3 = torch.cuda.Event(enable_timing=True)
                e3.record(stream)
                kev["fwd"].append((e0, e1))
                kev["bwd"].append((e2, e3))
            ops.bwd_finalize(dq_acc, scale, out=dq)
        dominant = "tile_bwd"
    else:
        dist.barrier()
        comm = GridComm(grid)
        if args.strategy == "ring":
            plan = RingAttention(comm, N, causal, scale)
        elif args.strategy == "attn2d_o":
            plan = Attention2DO(comm, N, causal, scale)
        else:
            plan = Attention2D(comm, N, causal, scale, head_chunks=args.head_chunks)
        q, k, v, do = (rnd((L, BH, H)) for _ in range(4))

        def step(record=False):
            o_p, saved = plan.forward(q, k, v)
            if not args.fwd_only:
                plan.backward(saved, do)
        dominant = "tile_bwd"

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    kev["fwd"].clear()
    kev["bwd"].clear()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ops.launches()
    ev0.record(stream)
    for _ in range(args.steps):
        step(record=True)
    ev1.record(stream)
    barrier()
    our_launches = ops.launches() - launches0
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = fl_step / (ms / 1e3) / 1e12

    peak_burst, peak_sus, hbm, peak_kind = measured_peaks()
    roof = None
    if kev["fwd"] and not kev["bwd"]:  # --fwd-only: the tile forward dominates
        kf = statistics.mean(a.elapsed_time(b) for a, b in kev["fwd"])
        ach = flops_fwd(B, M, H, N, causal) / (kf / 1e3) / 1e12
        roof = {"kernel": "tile_fwd (a2d_tile_fwd)", "bound": "tensor", "achieved": ach,
                "peak": peak_sus, "peak_kind": f"bf16_tflops_sustained ({peak_kind})",
                "unit": "TFLOP/s", "frac": ach / peak_sus, "traffic": None, "ms_per_launch": kf,
                "flops_per_launch": flops_fwd(B, M, H, N, causal)}
    if kev["bwd"]:
        kb = statistics.mean(a.elapsed_time(b) for a, b in kev["bwd"])
        kf = statistics.mean(a.elapsed_time(b) for a, b in kev["fwd"])
        ach = 2.5 * flops_fwd(B, M, H, N, causal) / (kb / 1e3) / 1e12
        roof = {"kernel": "tile_bwd (a2d_tile_bwd)", "bound": "tensor", "achieved": ach,
                "peak": peak_sus, "peak_kind": f"bf16_tflops_sustained ({peak_kind})",
                "unit": "TFLOP/s", "frac": ach / peak_sus, "traffic": None,
                "ms_per_launch": kb,
                "flops_per_launch": 2.5 * flops_fwd(B, M, H, N, causal),
                "other": {"tile_fwd": {"ms_per_launch": kf,
                                       "achieved": flops_fwd(B, M, H, N, causal) / (kf / 1e3) / 1e12,
                                       "frac": flops_fwd(B, M, H, N, causal) / (kf / 1e3) / 1e12
                                       / peak_sus}}}
        tp = ROOT / "profiles" / "traffic.json"
        if tp.exists():
            try:
                roof["traffic"] = json.loads(tp.read_text()).get("tile_bwd_bytes_per_launch")
            except ValueError:
                pass

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e and not args.fwd_only:
        # 1 GPU: functional.attention on [B, M, N, H]; N GPUs: each rank's shard
        # [N/P, B*M, H] (column-major cyclic / ring layout) through the
        # strategies' autograd entry point attention2d(q, k, v, plan)
        shape = (B, M, N, H) if world == 1 else (L, BH, H)
        if world > 1:
            from paper_2503_15758_b200.strategies import attention2d
        hosts = [torch.empty(shape, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
        for t in hosts:
            t.uniform_(-1, 1)
        res = torch.empty((1,), dtype=torch.float32).pin_memory()

        # Inputs of step i+1 are copied (pinned host -> HBM, copy stream) while
        # step i computes — a double-buffered input prefetcher, as a training
        # loop's data pipeline would run it; every step's copies and its loss
        # read-back stay inside the timed region.
        cs = torch.cuda.Stream(device=dev)
        bufs = [[torch.empty(shape, dtype=torch.bfloat16, device=dev) for _ in range(4)]
                for _ in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]

        def h2d(i):
            s_ = i % 2
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(done[s_])  # step i-2 has finished with these buffers
                for d_, h_ in zip(bufs[s_], hosts):
                    d_.copy_(h_, non_blocking=True)
                ready[s_].record(cs)

        def e2e_step(i, prefetch):
            s_ = i % 2
            stream.wait_event(ready[s_])
            if prefetch:
                h2d(i + 1)
            qd, kd, vd = (t.detach().requires_grad_(True) for t in bufs[s_][:3])
            dod = bufs[s_][3]
            if world == 1:
                out = functional.attention(qd, kd, vd, causal=causal, scale=scale)
            else:
                out = attention2d(qd, kd, vd, plan)
            out.backward(dod)
            # <O, dO> (the linearised loss whose gradient is dO), one fp32-accumulated dot
            loss = torch.dot(out.detach().reshape(-1), dod.reshape(-1)).float()
            res.copy_(loss.reshape(1), non_blocking=True)
            done[s_].record(stream)

        def run_steps(k):
            cs.wait_stream(stream)
            h2d(0)
            for i in range(k):
                e2e_step(i, i + 1 < k)

        run_steps(2)
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run_steps(args.steps)
        b.record(stream)
        barrier()
        ems = a.elapsed_time(b) / args.steps
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": fl_step / (ems / 1e3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": world * sum(t.numel() * t.element_size() for t in hosts),
               "d2h_bytes_per_step": 4 * world, "ms_per_step": ems,
               "path": ("paper_2503_15758_b200.functional.attention" if world == 1 else
                        f"paper_2503_15758_b200.strategies.attention2d ({args.strategy}, per-rank "
                        "shards)") + " (autograd); pinned host q/k/v/dO copied to HBM every step "
                       "on a copy stream (step i+1's copy overlaps step i's compute) and the loss "
                       "scalar read back; max over ranks"}
        del bufs
        del hosts

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_sample()

    if rank == 0:
        default = not (args.fwd_only or args.non_causal or args.grid) and N == 131072 and M == 32
        mode = f"{'causal' if causal else 'non-causal'} {'fwd' if args.fwd_only else 'fwd+bwd'}"
        line = {
            "metric": METRIC if default else f"attention {mode} TFLOP/s, N={N}, M={M}, H={H}",
            "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic uniform[-1,1] bf16 (torch.Generator on device)",
            "config": {"workload": f"exact {mode} attention, N={N}, M={M}, H={H}, B=1, "
                                   f"bf16, grid {grid.pr}x{grid.pc} ({args.strategy})",
                       "seq_len": N, "heads": M, "head_dim": H, "batch": B, "causal": causal,
                       "grid": f"{grid.pr}x{grid.pc}", "strategy": args.strategy,
                       "parallelism": f"2d{grid.pr}x{grid.pc}" if world > 1 else "1x1",
                       "flops_per_step": fl_step,
                       "l2": "every input is 1 GiB (> 126 MB L2); no flush needed"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": our_launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--strategy", choices=("attn2d_no", "attn2d_o", "ring"), default="attn2d_no")
    ap.add_argument("--seq-len", type=int, default=131072)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--head-chunks", type=int, default=4)
    ap.add_argument("--grid", default=None, help="Pr x Pc override, e.g. 4x2 (C5 sweep)")
    ap.add_argument("--fwd-only", action="store_true", help="forward only (C5 prefill)")
    ap.add_argument("--non-causal", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
