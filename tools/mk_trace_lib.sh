#!/bin/bash
# Build xlib/lib_TRACE.so: bwd128 with clock64 timestamps for one CTA (blockIdx TX,TY).
set -e
TX=${1:-3}; TY=${2:-5}
R=/root/repo/paper_2503_15758_b200/csrc
rm -rf /tmp/xt && mkdir -p /tmp/xt && cp $R/*.cu $R/*.cuh $R/*.h $R/Makefile /tmp/xt/
sed -i 's|../../include/attn2d_b200.h|/root/repo/include/attn2d_b200.h|' /tmp/xt/*
python3 - <<'PY'
p='/tmp/xt/tile_bwd128.cu'; s=open(p).read()
ev = [("const int qrow0 = cur.row0(p.q_map);", 0, 4, 'after'),
      ("mbar_wait(bar(B_QFULL0 + qs), (i >> 1) & 1);", 1, 4, 'before'),
      ("mbar_wait(bar(B_DOFULL), i & 1);", 2, 1, 'after'),
      ("mbar_wait(bar(B_PREADY), i & 1);", 3, 1, 'after'),
      ("mbar_wait(bar(B_DSREADY), i & 1);", 4, 1, 'after'),
      ("mbar_wait(bar(B_QFULL0 + (qs ^ 1)), ((i + 1) >> 1) & 1);", 5, 1, 'after'),
      ("mbar_wait(bar(B_DQFREE), (i - 1) & 1);", 6, 1, 'after'),
      ("mbar_wait(bar(B_QFULL0 + qs), (i >> 1) & 1);", 7, 4, 'after'),
      ("mbar_wait(bar(B_SFULL), i & 1);", 8, 4, 'after'),
      ("mbar_arrive(bar(B_PREADY));", 9, 4, 'before'),
      ("mbar_wait(bar(B_DPFULL), i & 1);", 10, 4, 'after'),
      ("if (i > 0) mbar_wait(bar(B_DSFREE), (i - 1) & 1);", 11, 4, 'after'),
      ("mbar_arrive(bar(B_DSREADY));", 12, 4, 'before'),
      ("mbar_wait(bar(B_DQFULL), i & 1);", 13, 12, 'after'),
      ("mbar_arrive(bar(B_DQFREE));", 14, 12, 'before'),
      ("bulk_commit_group();", 15, 12, 'after')]
# the same P/dS events for a warp of the second warpgroup (warp 8)
ev2 = [("mbar_arrive(bar(B_PREADY));", 16, 8, 'before'),
       ("mbar_arrive(bar(B_DSREADY));", 17, 8, 'before'),
       ("mbar_wait(bar(B_SFULL), i & 1);", 18, 8, 'after'),
       ("mbar_wait(bar(B_DPFULL), i & 1);", 19, 8, 'after')]
for pat, e, w, where in ev:
    assert pat in s, pat
    t = f"TRACE({e}, i, {w});"
    s = s.replace(pat, (pat + " " + t) if where == 'after' else (t + " " + pat), 1)
for pat, e, w, where in ev2:
    t = f"TRACE({e}, i, {w});"
    s = s.replace(pat, (pat + " " + t) if where == 'after' else (t + " " + pat), 1)
s = s.replace('#include "kernels.h"\n', '''#include "kernels.h"
__device__ long long g_trace[24][1024];
#define TRACE(ev, i, w) do { if (blockIdx.x == TX && blockIdx.y == TY && warp == (w) && (threadIdx.x & 31) == 0 && (i) < 1024) g_trace[ev][i] = clock64(); } while (0)
extern "C" int a2d_trace_dump(long long* host) { return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace)); }
''', 1)
open(p,'w').write(s)
PY
mkdir -p /root/repo/xlib2 && cd /tmp/xt && /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr -DTX=$TX -DTY=$TY $XFLAGS -shared -o /root/repo/xlib2/lib_TRACE$XSUF.so $(sed -n "s/^SRCS := //p" Makefile) -lcudart_static -lrt -ldl -lpthread
echo built
