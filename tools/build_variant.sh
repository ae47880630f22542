#!/bin/bash
# Build a variant of libhepkit_cuda.so with extra -D flags for one source
# (SRC=hk_fcn.cu by default; hk_phsp.cu / hk_sample.cu get -fmad=false as in
# the Makefile) into variants/<name>/libhepkit_cuda.so (select it with
# HK_LIB_PATH).  Used for A/B measurements of tuning macros; the product
# build is the Makefile's.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
SRC=${SRC:-hk_fcn.cu}
obj=${SRC%.cu}.o
B=paper_1711_05683_b200/csrc/build
EXTRA=""
case $SRC in hk_phsp.cu|hk_sample.cu) EXTRA="-fmad=false";; esac
mkdir -p variants/$name
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
  -Iinclude -Ipaper_1711_05683_b200/csrc --expt-relaxed-constexpr $EXTRA "$@" -c paper_1711_05683_b200/csrc/$SRC \
  -o variants/$name/$obj
objs=$(ls $B/*.o | grep -v "/$obj")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name/libhepkit_cuda.so \
  variants/$name/$obj $objs -lcudart -ldl
