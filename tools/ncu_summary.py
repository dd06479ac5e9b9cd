"""Summarise ncu captures for profiles/: launch-list shares and the key
counters of `ncu --set full` reports (read here, without a GPU).

usage: python tools/ncu_summary.py launches <launches.csv>
       python tools/ncu_summary.py report <x.ncu-rep> [algorithmic_flops_or_bytes] [unit]
       python tools/ncu_summary.py traffic <fwd.ncu-rep> <bwd.ncu-rep> <config> <commit> > profiles/traffic.json
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % of elapsed (tcgen05 utilisation)"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "shared-memory wavefronts to the tensor cores % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "shared-memory LSU wavefronts % of peak"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("dram__bytes.sum.per_second", "DRAM bandwidth"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed avg"),
    ("smsp__inst_executed.sum", "instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__sass_inst_executed_op_tmem_ldt.sum", "tcgen05.ld (LDTM)"),
    ("smsp__sass_inst_executed_op_tmem_stt.sum", "tcgen05.st (STTM)"),
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    tot = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0][:70]
        v = float(d["Metric Value"])
        unit = d["Metric Unit"]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                 "nsecond": 1e-6}.get(unit, 1e-6)
        t = tot.setdefault(name, [0.0, 0])
        t[0] += v * scale
        t[1] += 1
    s = sum(v[0] for v in tot.values())
    print("| kernel | launches | total ms | share |")
    print("|---|---|---|---|")
    for n, (v, c) in sorted(tot.items(), key=lambda x: -x[1][0]):
        print(f"| `{n}` | {c} | {v:.2f} | {100 * v / s:.1f}% |")


def report(path, algo=None, unit=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        print(f"### `{d.get('Kernel Name', '?').split('(')[0]}`\n")
        print("| counter | value |")
        print("|---|---|")
        for k, label in KEYS:
            if k in d:
                print(f"| {label} (`{k}`) | {d[k]} {u.get(k, '')} |")
        if algo:
            dur = float(d["gpu__time_duration.sum"])
            du = u.get("gpu__time_duration.sum", "ns")
            sec = dur * {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6,
                         "ms": 1e-3, "msecond": 1e-3}.get(du, 1e-9)
            print(f"| algorithmic {unit} per launch | {float(algo):.4g} |")
            print(f"| achieved (algorithmic / duration) | {float(algo) / sec / 1e12:.1f} T{unit}/s |")
        print()


def _raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[1])), [dict(zip(rows[0], r)) for r in rows[2:]]


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def traffic(fwd, bwd, config, commit):
    """DRAM bytes per launch (read + write) of the last captured launch of
    each report, for bench.py's roofline.traffic."""
    import json
    out = {"config": config, "source": f"ncu --set full --clock-control none, one launch each "
                                        f"(tools/perf_tile.py at {config}), commit {commit}"}
    for tag, path in (("tile_fwd", fwd), ("tile_bwd", bwd)):
        units, rows = _raw(path)
        r = rows[-1]
        total = sum(float(r[k]) * SCALE.get(units[k], 1)
                    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        out[f"{tag}_bytes_per_launch"] = int(total)
        k = "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"
        if k in r:
            out[f"{tag}_tensor_pipe_pct"] = float(r[k])
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(*sys.argv[2:6])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], *(sys.argv[3:5]))
