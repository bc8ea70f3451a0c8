#!/bin/bash
# Build libsparsh_b200.so variants with different compile-time knobs, in parallel:
#   tools/build_variants.sh NAME1 "-DFLAG=.." NAME2 "-DFLAG=.." ...
# -> _variants/NAME/libsparsh_b200.so (select with SB_LIB=...; tools only)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2007_00056_b200/csrc
L=$ROOT/paper_2007_00056_b200/_lib
make -C $CS >/dev/null
pids=()
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  d=$ROOT/_variants/$name; mkdir -p $d
  ( nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
      -fmad=false -I$ROOT/include $flags -c -o $d/sb_runtime.o $CS/sb_runtime.cu && \
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libsparsh_b200.so $L/sb_host.o $L/sb_dist.o $L/sb_galerkin.o $d/sb_runtime.o -lcudart -lpthread -ldl && \
    rm -f $d/sb_runtime.o && echo "built $name ($flags)" ) &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
