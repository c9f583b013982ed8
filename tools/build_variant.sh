#!/bin/bash
# Build a libzt.so variant with extra -D flags into build_var/<name>/libzt.so (experiments only)
# usage: tools/build_variant.sh NAME "-DFOO=1 -DBAR=2" [zt_oz.cu replacement]
set -e
cd "$(dirname "$0")/../paper_2206_05466_b200/csrc"
OUT=../../build_var/$1
mkdir -p $OUT
OZ=${3:-zt_oz.cu}
for f in zt_api zt_solve zt_gemm zt_basis; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $2 -c $f.cu -o $OUT/$f.o 2> $OUT/$f.ptxas.log &
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $2 -I. -x cu -c $OZ -o $OUT/zt_oz.o 2> $OUT/zt_oz.ptxas.log &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libzt.so $OUT/zt_api.o $OUT/zt_solve.o $OUT/zt_gemm.o $OUT/zt_basis.o $OUT/zt_oz.o -lcudart
grep -A2 k_oz_gemm $OUT/zt_oz.ptxas.log | grep -E "registers|spill" | tr '\n' ' '; echo
