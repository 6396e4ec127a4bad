#!/bin/bash
# Build experiment variants of libevo.so (EVO_EXP=n compile-time switches) into scripts/_exp/.
# Usage: scripts/build_exp.sh 1 2 3   -> scripts/_exp/libevo_exp{1,2,3}.so ; load with EVO_LIB_PATH=...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
P=$ROOT/paper_2203_00854_b200
for n in "$@"; do
  objs=""
  for f in $P/csrc/*.cu; do
    o=/tmp/exp${n}_$(basename $f .cu).o
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
      -I $ROOT/include -DEVO_EXP=$n ${EXTRA_FLAGS} -c $f -o $o &
    objs="$objs $o"
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared --cudart static -o $ROOT/scripts/_exp/libevo_exp$n.so $objs
  echo built scripts/_exp/libevo_exp$n.so
done
