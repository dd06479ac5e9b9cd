#!/bin/bash
# Build an experiment variant of the library: xlib/lib_<NAME>.so with extra -D flags.
# usage: tools/mk_xlib.sh NAME "-DFOO -DBAR"
set -e
NAME=$1; FL=$2
R=/root/repo/paper_2503_15758_b200/csrc
mkdir -p /root/repo/xlib
cd $R && /usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a \
  -Xcompiler -fPIC --expt-relaxed-constexpr $FL -shared -o /root/repo/xlib/lib_$NAME.so \
  $(sed -n "s/^SRCS := //p" Makefile) \
  -lcudart_static -lrt -ldl -lpthread
echo built xlib/lib_$NAME.so
