#!/bin/bash
# Round-end measurement set on one B200 (run under gpurun); outputs in gpurun_out/final_*
cd "$(dirname "$0")/.."
O=gpurun_out
make -C paper_2206_05466_b200/csrc -j8 > /dev/null
timeout 900 python -m pytest tests -m gpu -q > $O/final_gpu_tests.log 2>&1; echo "rc=$?" >> $O/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.log 2>&1
timeout 600 python bench.py > $O/final_bench.json 2> $O/final_bench.err
timeout 600 python bench.py --impl reference > $O/final_bench_ref.json 2>&1
ZT_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_oz_gemm -s 1 -c 1 \
  -o $O/final_oz_gemm python tools/oz_prof.py 2048 > /dev/null 2>&1
timeout 300 python tools/oz_zgemm_check.py > $O/final_oz_accuracy.txt 2>&1
timeout 900 python tools/cfg4_full.py > $O/final_cfg4_full.json 2>&1
timeout 600 python tools/bench_ops.py > $O/final_bench_ops.jsonl 2> $O/final_bench_ops.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solve_merged -c 2 \
  -o $O/final_solve python tools/solve_once.py 4096 1 > /dev/null 2>&1
