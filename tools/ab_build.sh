#!/bin/bash
# Build libgmx_exec.so from the exec sources of git revision $1 into _ab/$2/ (A/B experiments;
# _ab/ is git-ignored and travels with gpurun). usage: tools/ab_build.sh <rev> <name>
set -e
REV=$1; NAME=$2; D=_ab/$NAME; mkdir -p $D/src
for f in gmx_exec.cu gmx_runtime.cpp sm100_ptx.cuh; do git show $REV:paper_1901_10008_b200/csrc/exec/$f > $D/src/$f; done
mkdir -p $D/core; git show $REV:paper_1901_10008_b200/csrc/core/flatmap.hpp > $D/core/flatmap.hpp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -shared -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
  --expt-relaxed-constexpr -cudart static -I include -I paper_1901_10008_b200/csrc/exec $D/src/gmx_exec.cu $D/src/gmx_runtime.cpp \
  -o $D/libgmx_exec.so -L paper_1901_10008_b200/lib -lgmx_core -Xlinker -rpath,$PWD/paper_1901_10008_b200/lib -ldl
echo built $D/libgmx_exec.so
