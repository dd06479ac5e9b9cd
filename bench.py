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

`--gpus N` without torchrun launches N ranks itself (torch.distributed.run,
NCCL, 127.0.0.1) and fails if the node has fewer GPUs.  At N > 1 the same
invocation also times the same-kernel Ring Attention baseline and reports
`vs_ring` (ring.py:47-156).

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
REF = ROOT / "baseline" / "_ref"


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
# CPU legs: the reference itself (baseline/_ref) or its oracle port
# --------------------------------------------------------------------------

def _import_reference():
    """The unmodified reference package pip-installed into baseline/_ref
    (BASELINE.md §4), numpy kernel backend; None if it is not there."""
    if not (REF / "attn2d").is_dir():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/a2d_numba_cache")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    try:
        from attn2d import kernels
        from attn2d.attention import MaskKind
        from attn2d.strategies import DistAttnConfig, run_backward, run_forward
        from attn2d.strategies.common import Precision
    except ImportError:
        return None
    kernels.use_backend("numpy")
    return {"DistAttnConfig": DistAttnConfig, "run_forward": run_forward,
            "run_backward": run_backward, "MaskKind": MaskKind, "Precision": Precision}


def _c1_reference_seconds(ref) -> float:
    """BASELINE.json config 1 exactly: B=1, M=4, N=2048, H=64, fp32,
    non-causal forward on the simulated 2x2 grid, one head at a time
    (SPEC.md:389), through the reference's run_forward("attn2d_no")."""
    import numpy as np
    cfg = ref["DistAttnConfig"](n=2048, h=64, p=4, mask=ref["MaskKind"].NONE,
                                precision=ref["Precision"].SINGLE)
    rng = np.random.default_rng(0)
    t0 = time.perf_counter()
    for _ in range(4):
        q, k, v = (rng.uniform(-1, 1, (2048, 64)).astype(np.float32) for _ in range(3))
        ref["run_forward"]("attn2d_no", cfg, q, k, v)
    return time.perf_counter() - t0


def _cpu_model() -> str | None:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_sample(n_cpu=4096, h=128, causal=True, budget_s=12.0, max_heads=32, with_c1=True):
    """Time the reference algorithm on the host cores on a bounded sample of
    the metric workload: whole heads of N=n_cpu, causal fwd+bwd.  With the
    reference installed this is its own run_forward / run_backward
    ("attn2d_no", simulated 2x2 grid, numpy backend, float64); otherwise the
    oracle port of its numpy kernels."""
    import numpy as np
    ref = _import_reference()
    rng = np.random.default_rng(0)
    heads, t0 = 0, time.perf_counter()
    if ref is not None:
        cfg = ref["DistAttnConfig"](n=n_cpu, h=h, p=4,
                                    mask=ref["MaskKind"].CAUSAL if causal else ref["MaskKind"].NONE,
                                    scale=h ** -0.5)
        while heads < max_heads and (heads == 0 or time.perf_counter() - t0 < budget_s):
            q, k, v, do = (rng.uniform(-1, 1, (n_cpu, h)) for _ in range(4))
            fwd = ref["run_forward"]("attn2d_no", cfg, q, k, v)
            ref["run_backward"]("attn2d_no", cfg, fwd.saved, do)
            heads += 1
        kind = "reference"
        how = ("the reference's run_forward/run_backward('attn2d_no') on its simulated 2x2 grid "
               "(baseline/_ref attn2d 0.1.0, numpy backend, float64)")
    else:
        from oracle import attn2d_oracle as orc
        idx = np.arange(n_cpu)
        while heads < max_heads and (heads == 0 or time.perf_counter() - t0 < budget_s):
            q, k, v, do = (rng.uniform(-1, 1, (n_cpu, h)) for _ in range(4))
            o, lse, (m, d) = orc.tile_forward_full(q, k, v, idx, idx, causal, h ** -0.5, block=64)
            orc.tile_backward_full(q, k, v, o, do, m, d, idx, idx, causal, h ** -0.5)
            heads += 1
        kind = "port"
        how = "oracle port of kernels/numpy_backend.py (reference not installed), float64"
    dt = time.perf_counter() - t0
    fl = 3.5 * flops_fwd(1, heads, h, n_cpu, causal)
    out = {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": kind,
           "seconds": dt, "cpu_model": _cpu_model(),
           "backend": "numpy" if ref is not None else "oracle (numpy)",
           "sample": f"{heads} head(s) of N={n_cpu}, H={h}, {'causal' if causal else 'non-causal'} "
                     f"fwd+bwd through {how}; BLAS threads = all host cores"}
    if ref is not None and with_c1:
        out["c1_forward_seconds"] = _c1_reference_seconds(ref)
        out["c1"] = ("BASELINE.json config 1 exactly (B=1, M=4, N=2048, H=64, fp32, non-causal "
                     "forward, attn2d_no on the simulated 2x2 grid)")
    return out


def run_reference(args, rank):
    """--impl reference: the reference's CPU implementation on the host cores."""
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_sample(budget_s=0.0, max_heads=1, with_c1=False)
    vals = [cpu_sample(budget_s=0.0, max_heads=1, with_c1=False) for _ in range(args.steps)]
    v = statistics.median(x["value"] for x in vals)
    ms = statistics.median(x["seconds"] for x in vals) * 1e3
    cb = dict(vals[0])
    cb["value"] = v
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic uniform[-1,1]",
        "config": {"workload": "causal attention fwd+bwd, reference CPU implementation, bounded "
                               "sample of the N=131072 M=32 H=128 layer (1 head of N=4096 "
                               "per step)", "seq_len_sample": 4096, "heads_sample": 1,
                   "head_dim": 128, "causal": True},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# --------------------------------------------------------------------------
# kernel-interval accounting (the roofline of the dominant kernel at any N)
# --------------------------------------------------------------------------

_PAIRS: dict = {}


def _map_key(ti):
    if ti.is_array:
        return ("a", ti.n, id(ti.array))
    return ("f", ti.n, tuple(ti.bases), ti.stride, ti.rows_per_block)


def _pairs(qi, ki, nq, nk, causal) -> int:
    """Unmasked (q, k) pairs of one tile call (count_unmasked,
    attention.py:260-265), cached per index-map pair."""
    import numpy as np
    from paper_2503_15758_b200.ops import TokenIndex
    if not causal:
        return nq * nk
    qi = qi if qi is not None else TokenIndex.contiguous(nq)
    ki = ki if ki is not None else TokenIndex.contiguous(nk)
    key = (_map_key(qi), _map_key(ki))
    if key not in _PAIRS:
        _PAIRS[key] = int(np.searchsorted(np.sort(ki.host()), qi.host(), side="right").sum())
    return _PAIRS[key]


class TimedCompute:
    """Proxy over the kernel module handed to a strategy plan: records a
    (start, end) marker pair on the launching stream around every tile
    forward / backward launch, with the launch's algorithmic FLOPs."""

    def __init__(self, inner, mark):
        self.inner = inner
        self.mark = mark
        self.records: list = []
        self.on = False

    def __getattr__(self, name):
        return getattr(self.inner, name)

    def _timed(self, kind, fn, flops, *a, **k):
        if not self.on:
            return fn(*a, **k)
        m0 = self.mark()
        r = fn(*a, **k)
        self.records.append((kind, m0, self.mark(), flops))
        return r

    def tile_forward(self, q, k, v, **kw):
        fl = 4.0 * q.shape[0] * q.shape[2] * _pairs(kw.get("q_index"), kw.get("k_index"),
                                                     q.shape[1], k.shape[1], kw["causal"])
        return self._timed("fwd", self.inner.tile_forward, fl, q, k, v, **kw)

    def tile_backward(self, q, k, v, dout, lse, delta, **kw):
        fl = 10.0 * q.shape[0] * q.shape[2] * _pairs(kw.get("q_index"), kw.get("k_index"),
                                                      q.shape[1], k.shape[1], kw["causal"])
        return self._timed("bwd", self.inner.tile_backward, fl, q, k, v, dout, lse, delta, **kw)

    def summary(self, elapsed, steps: int) -> dict:
        out = {}
        for kind in ("fwd", "bwd"):
            rec = [(elapsed(a, b), f) for kd, a, b, f in self.records if kd == kind]
            if rec:
                ms = sum(r[0] for r in rec)
                fl = sum(r[1] for r in rec)
                out[kind] = {"ms_per_step": ms / steps, "launches_per_step": len(rec) / steps,
                             "flops_per_step": fl / steps, "tflops": fl / (ms / 1e3) / 1e12}
        return out


def cuda_marks(stream_fn):
    import torch

    def mark():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream_fn())
        return e
    return mark, (lambda a, b: a.elapsed_time(b))


def cpu_marks():
    return time.perf_counter, (lambda a, b: (b - a) * 1e3)


def make_plan(strategy, comm, n, causal, scale, head_chunks, compute):
    from paper_2503_15758_b200.strategies import Attention2D, Attention2DO, RingAttention
    if strategy == "ring":
        return RingAttention(comm, n, causal, scale, compute=compute)
    if strategy == "attn2d_o":
        return Attention2DO(comm, n, causal, scale, compute=compute)
    return Attention2D(comm, n, causal, scale, head_chunks=head_chunks, compute=compute)


def run_dist(args, rank, world, dev, compute, mark, elapsed, sync, dtype=None):
    """The N > 1 measurement, device-agnostic (NCCL + CUDA events on the
    B200 box; gloo + the CPU stand-in in tests/test_bench_contract.py):
    times `--strategy` and, unless --no-ring, the same-kernel Ring baseline,
    over per-rank shards [N/P, B*M, H].  Returns a dict of per-rank
    measurements (ms are this rank's; the caller takes the max)."""
    import torch
    import torch.distributed as dist
    from paper_2503_15758_b200.layouts import Grid2D
    from paper_2503_15758_b200.strategies import GridComm

    N, M, H = args.seq_len, args.heads, args.head_dim
    causal = not args.non_causal
    scale = H ** -0.5
    pr, pc = GRIDS.get(world, (1, world))
    if args.grid:
        pr, pc = (int(x) for x in args.grid.lower().split("x"))
        if pr * pc != world:
            raise SystemExit(f"--grid {args.grid} does not match {world} ranks")
    L = N // world
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    dtype = dtype or torch.bfloat16
    q, k, v, do = (torch.empty((L, M, H), dtype=torch.float32, device=dev)
                   .uniform_(-1, 1, generator=g).to(dtype) for _ in range(4))
    res = {"grid": f"{pr}x{pc}"}

    def measure(strategy, grid):
        comm = GridComm(grid)
        timed = TimedCompute(compute, mark)
        plan = make_plan(strategy, comm, N, causal, scale, args.head_chunks, timed)

        def step():
            o_p, saved = plan.forward(q, k, v)
            if not args.fwd_only:
                plan.backward(saved, do)
        for _ in range(args.warmup):
            step()
        sync()
        dist.barrier()
        comm.ledger.rows.clear()
        timed.on = True
        m0 = mark()
        for _ in range(args.steps):
            step()
        m1 = mark()
        sync()
        dist.barrier()
        timed.on = False
        ms = elapsed(m0, m1) / args.steps
        led = comm.ledger
        return {"ms": ms, "plan": plan, "kernels": timed.summary(elapsed, args.steps),
                "bytes_out_per_step": led.bytes_out() / args.steps,
                "msgs_per_step": led.msgs_out() / args.steps,
                "ledger": led.as_dict()}

    main_grid = Grid2D(pr, pc) if args.strategy in ("attn2d_no", "attn2d_o") else Grid2D(1, world)
    res["main"] = measure(args.strategy, main_grid)
    if not args.no_ring and args.strategy != "ring":
        res["ring"] = measure("ring", Grid2D(1, world))
    return res


def _max_over_ranks(x: float, dev) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_line_fields(args, res, world, dev, peak):
    """Contract fields of the N > 1 line from run_dist's per-rank results
    (max over ranks for every time; the kernel roofline is the slowest
    rank's dominant kernel)."""
    import torch.distributed as dist
    causal = not args.non_causal
    fl_step = (1.0 if args.fwd_only else 3.5) * flops_fwd(1, args.heads, args.head_dim,
                                                          args.seq_len, causal)
    ms = _max_over_ranks(res["main"]["ms"], dev)
    out = {"ms_per_step": ms, "value": fl_step / (ms / 1e3) / 1e12, "flops_per_step": fl_step}
    kind = "fwd" if args.fwd_only else "bwd"
    ker = res["main"]["kernels"].get(kind)
    allk = [None] * world
    dist.all_gather_object(allk, res["main"]["kernels"])
    if ker:
        worst = min((k[kind]["tflops"], i) for i, k in enumerate(allk) if kind in k)
        k0 = allk[worst[1]][kind]
        out["roofline"] = {
            "kernel": f"tile_{kind} (a2d_tile_{kind})", "bound": "tensor",
            "achieved": k0["tflops"], "peak": peak[1],
            "peak_kind": f"bf16_tflops_sustained ({peak[3]})", "unit": "TFLOP/s",
            "frac": k0["tflops"] / peak[1], "traffic": None, "rank": worst[1],
            "ms_per_step": k0["ms_per_step"], "flops_per_step_rank": k0["flops_per_step"],
            "launches_per_step": k0["launches_per_step"],
            "per_rank_tflops": [k[kind]["tflops"] if kind in k else None for k in allk],
            "share_of_step": k0["ms_per_step"] / ms}
    byt = [None] * world
    dist.all_gather_object(byt, (res["main"]["bytes_out_per_step"],
                                 res["main"]["msgs_per_step"]))
    out["comm"] = {"bytes_out_per_rank_per_step_max": max(b[0] for b in byt),
                   "messages_per_rank_per_step_max": max(b[1] for b in byt),
                   "ledger_rank0": res["main"]["ledger"], "transport": "torch.distributed"}
    if "ring" in res:
        rms = _max_over_ranks(res["ring"]["ms"], dev)
        rv = fl_step / (rms / 1e3) / 1e12
        rb = [None] * world
        dist.all_gather_object(rb, res["ring"]["bytes_out_per_step"])
        out["ring"] = {"value": rv, "ms_per_step": rms, "unit": "TFLOP/s",
                       "bytes_out_per_rank_per_step_max": max(rb),
                       "strategy": "ring (same tile kernels, ring.py:47-156)"}
        out["vs_ring"] = out["value"] / rv
    return out


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2503_15758_b200 import _lib, functional, ops

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    _lib.load()
    N, M, H, B = args.seq_len, args.heads, args.head_dim, 1
    BH = B * M
    causal = not args.non_causal
    scale = H ** -0.5
    fl_step = (1.0 if args.fwd_only else 3.5) * flops_fwd(B, M, H, N, causal)
    stream = torch.cuda.current_stream()
    peak = measured_peaks()
    kev = {"bwd": [], "fwd": []}
    dist_fields = None

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local_rank)
    if world == 1:
        g = torch.Generator(device=dev).manual_seed(1234)

        def rnd(shape):
            return torch.empty(shape, dtype=torch.bfloat16, device=dev).uniform_(-1, 1,
                                                                                  generator=g)
        q, k, v, do = (rnd((BH, N, H)) for _ in range(4))
        dq_acc = torch.zeros((BH, N, H), dtype=torch.float32, device=dev)
        o = torch.empty_like(q)
        lse = torch.empty((BH, N), dtype=torch.float32, device=dev)
        dk, dv = torch.empty_like(k), torch.empty_like(v)
        dq = torch.empty_like(q)

        def step(record=False):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if record else None
            if record:
                ev[0].record(stream)
            ops.tile_forward(q, k, v, causal=causal, scale=scale, out=o, lse=lse,
                             out_dtype=torch.bfloat16)
            if record:
                ev[1].record(stream)
                kev["fwd"].append((ev[0], ev[1]))
            if args.fwd_only:
                return
            delta = ops.bwd_preprocess(o, do)
            dq_acc.zero_()
            if record:
                ev[2].record(stream)
            ops.tile_backward(q, k, v, do, lse, delta, causal=causal, scale=scale, dq_acc=dq_acc,
                              dk=dk, dv=dv)
            if record:
                ev[3].record(stream)
                kev["bwd"].append((ev[2], ev[3]))
            ops.bwd_finalize(dq_acc, scale, out=dq)

        for _ in range(args.warmup):
            step()
        barrier()
        sampler.start()
        time.sleep(0.3)
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
        value = fl_step / (ms / 1e3) / 1e12
    else:
        mark, elapsed = cuda_marks(lambda: torch.cuda.current_stream())
        dist.barrier()
        sampler.start()
        time.sleep(0.3)
        launches0 = ops.launches()
        res = run_dist(args, rank, world, dev, ops, mark, elapsed, torch.cuda.synchronize)
        our_launches = ops.launches() - launches0
        clocks = sampler.stop()
        dist_fields = dist_line_fields(args, res, world, dev, peak)
        ms, value = dist_fields["ms_per_step"], dist_fields["value"]
        plan = res["main"]["plan"]

    roof = None
    if world == 1 and kev["fwd"]:
        kf = statistics.mean(a.elapsed_time(b) for a, b in kev["fwd"])
        ff = flops_fwd(B, M, H, N, causal)
        fwd_info = {"ms_per_launch": kf, "achieved": ff / (kf / 1e3) / 1e12,
                    "frac": ff / (kf / 1e3) / 1e12 / peak[1]}
        if not kev["bwd"]:
            roof = {"kernel": "tile_fwd (a2d_tile_fwd)", "bound": "tensor",
                    "achieved": fwd_info["achieved"], "peak": peak[1],
                    "peak_kind": f"bf16_tflops_sustained ({peak[3]})", "unit": "TFLOP/s",
                    "frac": fwd_info["frac"], "traffic": None, "ms_per_launch": kf,
                    "flops_per_launch": ff}
        else:
            kb = statistics.mean(a.elapsed_time(b) for a, b in kev["bwd"])
            ach = 2.5 * ff / (kb / 1e3) / 1e12
            roof = {"kernel": "tile_bwd (a2d_tile_bwd)", "bound": "tensor", "achieved": ach,
                    "peak": peak[1], "peak_kind": f"bf16_tflops_sustained ({peak[3]})",
                    "unit": "TFLOP/s", "frac": ach / peak[1], "traffic": None,
                    "ms_per_launch": kb, "flops_per_launch": 2.5 * ff,
                    "share_of_step": kb / ms, "other": {"tile_fwd": fwd_info}}
        tp = ROOT / "profiles" / "traffic.json"
        if tp.exists():
            try:
                t = json.loads(tp.read_text())
                key = "tile_fwd_bytes_per_launch" if args.fwd_only else "tile_bwd_bytes_per_launch"
                if t.get("config") == f"N={N} M={M} H={H} causal={int(causal)}" and key in t:
                    roof["traffic"] = t[key]
                    roof["traffic_source"] = t.get("source")
            except ValueError:
                pass
    elif dist_fields is not None:
        roof = dist_fields.get("roofline")

    # ---------------------------------------------------------------- e2e
    e2e = None
    e2e_train = None
    if not args.no_e2e and not args.fwd_only:
        e2e, e2e_train = run_e2e(args, world, dev, stream, barrier, fl_step,
                                 plan if world > 1 else None)

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_sample()

    parity = None
    pp = ROOT / "profiles" / "parity.json"
    if pp.exists():
        try:
            pj = json.loads(pp.read_text())
            parity = {"source": "profiles/parity.json (tools/parity_report.py)",
                      "reference": pj.get("reference"), "commit": pj.get("commit"),
                      "worst": pj.get("worst"),
                      "rel_fro": {c: {t: round(e["rel_fro"], 6) for t, e in v["errors"].items()}
                                  for c, v in pj.get("configs", {}).items()}}
        except (ValueError, KeyError):
            parity = None

    if rank == 0:
        default = (not (args.fwd_only or args.non_causal or args.grid) and N == 131072
                   and M == 32 and H == 128)
        mode = f"{'causal' if causal else 'non-causal'} {'fwd' if args.fwd_only else 'fwd+bwd'}"
        gname = dist_fields and res["grid"] or "1x1"
        line = {
            "metric": METRIC if default else f"attention {mode} TFLOP/s, N={N}, M={M}, H={H}",
            "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic uniform[-1,1] bf16 (torch.Generator on device)",
            "config": {"workload": f"exact {mode} attention, N={N}, M={M}, H={H}, B=1, "
                                   f"bf16, grid {gname} ({args.strategy})",
                       "seq_len": N, "heads": M, "head_dim": H, "batch": B, "causal": causal,
                       "grid": gname, "strategy": args.strategy,
                       "parallelism": f"2d{gname}" if world > 1 else "1x1",
                       "flops_per_step": fl_step,
                       "l2": "every input is >= 128 MiB per rank (> 126 MB L2); no flush needed"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "e2e_training_step": e2e_train,
            "gpu_launches": our_launches, "clocks": clocks, "parity": parity,
        }
        if dist_fields is not None:
            for key in ("vs_ring", "ring", "comm"):
                if key in dist_fields:
                    line[key] = dist_fields[key]
        print(json.dumps(line), flush=True)


def run_e2e(args, world, dev, stream, barrier, fl_step, plan):
    """The same metric through the public API with host buffers: every step
    copies its q/k/v/dO from pinned host memory (H2D) and its results back
    (D2H).  `e2e` returns the reference API's outputs to the host — O, dQ,
    dK, dV (the reference's run_forward / run_backward return host arrays);
    `e2e_training_step` reads back only the loss scalar.  Step i+1's inputs
    are copied while step i computes, and step i's results are read back
    while step i+1 computes (copy engines on their own streams); all copies
    of the timed steps are inside the timed region."""
    import torch
    import torch.distributed as dist
    from paper_2503_15758_b200 import functional

    N, M, H = args.seq_len, args.heads, args.head_dim
    causal = not args.non_causal
    scale = H ** -0.5
    shape = (1, M, N, H) if world == 1 else (N // world, M, H)
    if world > 1:
        from paper_2503_15758_b200.strategies import attention2d
    hosts = [torch.empty(shape, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
    for t in hosts:
        t.uniform_(-1, 1)
    outs_h = [[torch.empty(shape, dtype=torch.bfloat16).pin_memory() for _ in range(4)]
              for _ in range(2)]
    loss_h = torch.empty((2,), dtype=torch.float32).pin_memory()
    cs_in = torch.cuda.Stream(device=dev)
    cs_out = torch.cuda.Stream(device=dev)
    bufs = [[torch.empty(shape, dtype=torch.bfloat16, device=dev) for _ in range(4)]
            for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    copied = [torch.cuda.Event() for _ in range(2)]
    results: list = [None, None]

    def h2d(i):
        s_ = i % 2
        with torch.cuda.stream(cs_in):
            if i >= 2:
                cs_in.wait_event(done[s_])  # step i-2 has finished with these buffers
            for d_, h_ in zip(bufs[s_], hosts):
                d_.copy_(h_, non_blocking=True)
            ready[s_].record(cs_in)

    def d2h(i, full):
        s_ = i % 2
        with torch.cuda.stream(cs_out):
            cs_out.wait_event(done[s_])
            if full:
                for h_, t in zip(outs_h[s_], results[s_]):
                    t.record_stream(cs_out)  # the allocator must not recycle it mid-copy
                    h_.copy_(t, non_blocking=True)
            copied[s_].record(cs_out)

    def e2e_step(i, prefetch, full):
        s_ = i % 2
        stream.wait_event(ready[s_])
        if i >= 2:
            stream.wait_event(copied[s_])  # results of step i-2 have left these tensors
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
        loss_h[s_:s_ + 1].copy_(loss.reshape(1), non_blocking=True)
        results[s_] = (out.detach(), qd.grad, kd.grad, vd.grad)
        done[s_].record(stream)
        d2h(i, full)

    def run_steps(k, full):
        cs_in.wait_stream(stream)
        h2d(0)
        for i in range(k):
            e2e_step(i, i + 1 < k, full)

    def timed(full):
        run_steps(2, full)
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run_steps(args.steps, full)
        stream.wait_stream(cs_out)
        b.record(stream)
        barrier()
        ems = a.elapsed_time(b) / args.steps
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        return ems

    per = sum(t.numel() * t.element_size() for t in hosts)
    ems = timed(True)
    e2e = {"value": fl_step / (ems / 1e3) / 1e12, "unit": "TFLOP/s",
           "h2d_bytes_per_step": world * per, "d2h_bytes_per_step": world * (per + 4),
           "ms_per_step": ems,
           "path": ("paper_2503_15758_b200.functional.attention" if world == 1 else
                    f"paper_2503_15758_b200.strategies.attention2d ({args.strategy}, per-rank "
                    "shards)") + " (autograd); every step: pinned host q/k/v/dO -> HBM and "
                   "O/dQ/dK/dV + loss -> pinned host, copies overlapped with the neighbouring "
                   "steps' compute on copy streams; max over ranks"}
    ems_t = timed(False)
    e2e_t = {"value": fl_step / (ems_t / 1e3) / 1e12, "unit": "TFLOP/s",
             "h2d_bytes_per_step": world * per, "d2h_bytes_per_step": world * 4,
             "ms_per_step": ems_t, "path": "as e2e, reading back only the loss scalar"}
    return e2e, e2e_t


def _self_launch(args) -> int:
    """--gpus N > 1 outside torchrun: one rank per GPU over NCCL."""
    import socket

    import torch
    n = torch.cuda.device_count()
    if args.impl == "ours" and n < args.gpus:
        raise SystemExit(f"--gpus {args.gpus} needs {args.gpus} CUDA devices, this node has {n}")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--strategy", choices=("attn2d_no", "attn2d_o", "ring"), default="attn2d_no")
    ap.add_argument("--seq-len", type=int, default=131072)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--head-chunks", type=int, default=4)
    ap.add_argument("--grid", default=None, help="Pr x Pc override, e.g. 4x2 (C5 sweep)")
    ap.add_argument("--fwd-only", action="store_true", help="forward only (C5 prefill)")
    ap.add_argument("--non-causal", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ring", action="store_true", help="N>1: skip the same-kernel Ring arm")
    return ap.parse_args(argv)


def main():
    args = parse_args()
    if args.warmup < 0 or args.steps < 1:
        raise SystemExit("need --steps >= 1 and --warmup >= 0")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "reference":  # the CPU arm runs on rank 0 only
            run_reference(args, 0)
            return
        raise SystemExit(_self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and args.impl == "ours":
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
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
