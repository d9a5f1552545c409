#!/bin/bash
# Build a variant of libparm_b200.so with extra -D flags into tools/probes/variants/<name>.so
#   bash tools/probes/build_variant.sh <name> "-DFOO=1 -DBAR=2"
set -e
name=$1; defs=$2
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
out=$ROOT/tools/probes/variants; mkdir -p $out/$name
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I $ROOT/include $defs"
objs=""
for s in capi gate permute gemm_sm100; do
  nvcc $F -c $ROOT/paper_2407_00599_b200/csrc/$s.cu -o $out/$name/$s.o &
  objs="$objs $out/$name/$s.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/$name.so $objs
echo $out/$name.so
