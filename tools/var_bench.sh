#!/bin/bash
# Step time of the in-tree library and build_var/<name> variants (experiments):
# usage: tools/var_bench.sh NAME ...   ("default" = paper_2206_05466_b200/libzt.so)
for v in "$@"; do
  if [ "$v" = default ]; then L=$PWD/paper_2206_05466_b200/libzt.so; else L=$PWD/build_var/$v/libzt.so; fi
  echo -n "$v "
  ZT_LIB_PATH=$L timeout 300 python bench.py --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), round(d['value'],1), d['clocks']['sm_mhz'])"
done
