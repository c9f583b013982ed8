#!/bin/bash
# Step time under environment settings (experiments): usage tools/env_bench.sh "ENV=.." "ENV=.." ...
for e in "$@"; do
  echo -n "$e "
  env $e timeout 300 python bench.py --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
done
