#!/bin/bash
# Build a libzt.so variant with extra -D flags into build_var/<name>.so (experiments only)
# usage: tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
cd "$(dirname "$0")/../paper_2206_05466_b200/csrc"
OUT=../../build_var/$1
mkdir -p $OUT
for f in zt_api zt_solve zt_gemm zt_basis zt_oz; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $2 -c $f.cu -o $OUT/$f.o 2> $OUT/$f.ptxas.log &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libzt.so $OUT/zt_api.o $OUT/zt_solve.o $OUT/zt_gemm.o $OUT/zt_basis.o $OUT/zt_oz.o -lcudart
grep -A2 k_solve_merged $OUT/zt_solve.ptxas.log | grep -E "registers|spill" | tr '\n' ' '; echo
