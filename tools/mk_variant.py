"""Build A/B variants of the library from patched copies of csrc/ (the product
sources stay free of experiment switches).

    python tools/mk_variant.py NAME [NAME ...]      -> xlib2/lib_NAME.so
    A2D_LIB_PATH=xlib2/lib_NAME.so python tools/perf_tile.py bwd 32768 32 128 1

Each variant is a list of (file, old, new) string replacements; an `old`
that is not found aborts the build.  xlib2/ is scratch (git-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_2503_15758_b200" / "csrc"
OUT = ROOT / "xlib2"

B = "tile_bwd128.cu"
F = "tile_fwd2.cu"
VARIANTS: dict[str, list[tuple[str, str, str]]] = {
    "base": [],
    # upper bound: no dQ reduce at all (wrong results)
    "nodq": [(B, "          tma_reduce_add_3d_g(&tm_dq, buf, 0, qrow + DQ_ROWS * r, bh);",
              "          if (false) tma_reduce_add_3d_g(&tm_dq, buf, 0, qrow + DQ_ROWS * r, bh);")],
    # half the dQ bytes (wrong results)
    "halfdq": [(B, "          tma_reduce_add_3d_g(&tm_dq, buf, 0, qrow + DQ_ROWS * r, bh);",
                "          if (r < DQ_ROUNDS / 2) tma_reduce_add_3d_g(&tm_dq, buf, 0, qrow + DQ_ROWS * r, bh);")],
    # half the staging bytes in flight (2 x 8 KB instead of 4 x 8 KB)
    "stage16k": [(B, "constexpr int DQ_BUFS = 4;\nconstexpr int DQ_ROWS = 64 / DQ_BUFS;",
                  "constexpr int DQ_BUFS = 2;\nconstexpr int DQ_ROWS = 16;")],
    # TMA tensor STORE instead of reduce-add (wrong results): the L2 RMW cost
    "dqstore": [(B, "          tma_reduce_add_3d_g(&tm_dq, buf, 0, qrow + DQ_ROWS * r, bh);",
                 "          asm volatile(\"cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group"
                 " [%0, {%2, %3, %4}], [%1];\" :: \"l\"(reinterpret_cast<uint64_t>(&tm_dq)),"
                 " \"r\"(buf), \"r\"(0), \"r\"(qrow + DQ_ROWS * r), \"r\"(bh) : \"memory\");")],
    # no wait for the staging buffer's previous reduce (races, wrong results)
    "dqnowait": [(B, "        if (h == 0) bulk_wait_group_read<DQ_BUFS - 1>();", "")],
    # forward: a quarter of the exponential pairs on the FMA polynomial
    "fpoly4": [(F, "#define F2_POLY(jj) ((((jj) >> 1) & 7) == 7)", "#define F2_POLY(jj) ((((jj) >> 1) & 3) == 3)")],
    "fpoly0": [(F, "#define F2_POLY(jj) ((((jj) >> 1) & 7) == 7)", "#define F2_POLY(jj) false")],
    # dQ = dS K (TMEM lane = query row) drained by 16-byte red.global.add.v4.f32
    # straight from registers: no shared-memory staging, no TMA reduce
    "dqred4": [
        (B, "umma_bf16(tmem + TM_Y, kb + mofs(kk), dsb + mofs(kk), id_mnmn, kk > 0);",
            "umma_bf16(tmem + TM_Y, dsb + mofs(kk), kb + mofs(kk), id_mnmn, kk > 0);"),
        (B, """#pragma unroll
      for (int r = 0; r < DQ_ROUNDS; ++r) {
        const uint32_t buf = sb + OFF_DQ + (round % DQ_BUFS) * DQ_BUF_BYTES;""",
            """const TileRef qtl = tile_ref(p.q_map, p.nq, qrow);
      if (h < qtl.nvalid) {
        float* dst = p.dq_acc + (long long)bh * p.dq_stride_bh + (long long)(qrow + h) * p.dq_stride_row;
#pragma unroll
        for (int c = 0; c < 128; c += 4)
          if (c < p.h)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(dst + c),
                         "f"(v[c]), "f"(v[c + 1]), "f"(v[c + 2]), "f"(v[c + 3]) : "memory");
      }
#pragma unroll
      for (int r = 0; r < 0; ++r) {
        const uint32_t buf = sb + OFF_DQ + (round % DQ_BUFS) * DQ_BUF_BYTES;"""),
    ],
    # no dQ drain work at all besides reading TMEM (wrong results): SMEM bound test
    "nodqsts": [(B, "for (int r = 0; r < DQ_ROUNDS; ++r) {", "for (int r = 0; r < 0; ++r) {")],
    # clock64 timeline of forward CTA (3, 5) for tools/trace_fwd2.py
    "ftrace": [(F, "// clock64 instrumentation points;", "#define A2D_TRACE 1\n#define TX 3\n#define TY 5\n// clock64 instrumentation points;")],
    # backward: every mbarrier wait suspend-hinted instead of spinning
    "bwdsleep": [(B, "#include \"kernels.h\"", "#include \"kernels.h\"\n#define mbar_wait mbar_wait_sleep")],
    # forward: the softmax warps' S-ready waits suspend-hinted too
    "fwdsleep": [(F, "#include \"kernels.h\"", "#include \"kernels.h\"\n#define mbar_wait mbar_wait_sleep")],
    # forward: the two softmax warpgroups take turns in the exponential phase
    # (named barriers 2/3, 256 threads): no MUFU sharing between the tiles
    "fpp": [(F, "      float tsum = exps(m_run == -INFINITY ? 0.f : m_run);",
             "      named_bar_sync(2 + t, 256);\n"
             "      float tsum = exps(m_run == -INFINITY ? 0.f : m_run);\n"
             "      named_bar_arrive(3 - t, 256);"),
            (F, "    const TileRef qt = t ? qt1 : qt0;\n    for (int j = 0; j < n_tiles; ++j) {",
             "    const TileRef qt = t ? qt1 : qt0;\n    if (t == 1 && n_tiles > 0) named_bar_arrive(2, 256);\n"
             "    for (int j = 0; j < n_tiles; ++j) {"),
            (F, "    // ------------------------------------------------------------ epilogue\n    if (n_tiles > 0) {",
             "    // ------------------------------------------------------------ epilogue\n"
             "    if (t == 0 && n_tiles > 0) named_bar_sync(2, 256);\n    if (n_tiles > 0) {")],
}


# (bound, wrong results) Q / dO tiles loaded by TMA only for the first two
# query tiles: what the per-SM TMA engine's load work costs the backward
VARIANTS["noqload"] = [
    (B, """            mbar_expect_tx(bar(B_QFULL0 + qs), TILE_B);
            for (int s = 0; s < 2; ++s)""", """            mbar_expect_tx(bar(B_QFULL0 + qs), i < 2 ? TILE_B : 0);
            for (int s = 0; s < 2 && i < 2; ++s)"""),
    (B, """            mbar_expect_tx(bar(B_DOFULL), TILE_B);
            for (int s = 0; s < 2; ++s)""", """            mbar_expect_tx(bar(B_DOFULL), i < 2 ? TILE_B : 0);
            for (int s = 0; s < 2 && i < 2; ++s)"""),
]
# (bound, wrong results) only the dO loads skipped
VARIANTS["nodoload"] = VARIANTS["noqload"][1:]

# dQ staging: 3 x 8 KB (frees 8 KB of shared memory)
VARIANTS["stage24k"] = [(B, "constexpr int DQ_BUFS = 4;\nconstexpr int DQ_ROWS = 64 / DQ_BUFS;",
                         "constexpr int DQ_BUFS = 3;\nconstexpr int DQ_ROWS = 16;")]
VARIANTS["fpp4"] = VARIANTS["fpp"] + VARIANTS["fpoly4"]
VARIANTS["fpptrace"] = VARIANTS["fpp"] + VARIANTS["ftrace"]


def build(name: str) -> Path:
    patches = VARIANTS[name]
    work = Path("/tmp") / f"a2d_var_{name}"
    if work.exists():
        shutil.rmtree(work)
    shutil.copytree(CSRC, work / "pkg" / "csrc", ignore=shutil.ignore_patterns("build"))
    shutil.copytree(ROOT / "include", work / "include")
    rev = os.environ.get("REV")  # sources of a git revision instead of the work tree
    if rev:
        for f in (work / "pkg" / "csrc").iterdir():
            if f.is_file():
                rel = f"paper_2503_15758_b200/csrc/{f.name}"
                out = subprocess.run(["git", "show", f"{rev}:{rel}"], cwd=ROOT,
                                     capture_output=True)
                if out.returncode == 0:
                    f.write_bytes(out.stdout)
        hdr = subprocess.run(["git", "show", f"{rev}:include/attn2d_b200.h"], cwd=ROOT,
                             capture_output=True, check=True).stdout
        (work / "include" / "attn2d_b200.h").write_bytes(hdr)
    for fname, old, new in patches:
        p = work / "pkg" / "csrc" / fname
        s = p.read_text()
        if old not in s:
            raise SystemExit(f"{name}: patch target not found in {fname}: {old[:60]!r}")
        p.write_text(s.replace(old, new))
    OUT.mkdir(exist_ok=True)
    lib = OUT / f"lib_{name}{os.environ.get('SUFFIX', '')}.so"
    mk = work / "pkg" / "csrc" / "Makefile"
    mk.write_text(mk.read_text().replace("LIB := ../libattn2d_b200.so", f"LIB := {lib}"))
    subprocess.run(["make", "-C", str(work / "pkg" / "csrc"), "-j8", "-s"], check=True)
    return lib


if __name__ == "__main__":
    for n in sys.argv[1:] or list(VARIANTS):
        print("built", build(n))
