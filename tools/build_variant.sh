#!/bin/bash
# Build a variant of libhepkit_cuda.so with extra -D flags for hk_fcn.cu into
# variants/<name>/libhepkit_cuda.so (select it with HK_LIB_PATH).  Used for
# A/B measurements of tuning macros; the product build is the Makefile's.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
B=paper_1711_05683_b200/csrc/build
mkdir -p variants/$name
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
  -Iinclude -Ipaper_1711_05683_b200/csrc --expt-relaxed-constexpr "$@" -c paper_1711_05683_b200/csrc/hk_fcn.cu \
  -o variants/$name/hk_fcn.o
objs=$(ls $B/*.o | grep -v hk_fcn.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name/libhepkit_cuda.so \
  variants/$name/hk_fcn.o $objs -lcudart -ldl
