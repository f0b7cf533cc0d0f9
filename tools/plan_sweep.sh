#!/bin/bash
# Bench the cfg3 fused solve under planner overrides (cluster size / columns per thread).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in ${SWEEP_C:-2 4 8 16}; do for lc in ${SWEEP_LC:-1 2 4 8 16}; do
  r=$(DDB_PLAN_C=$c DDB_PLAN_LC=$lc timeout 120 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-latency ${BENCH_ARGS} 2>/dev/null | tail -1)
  echo "C=$c LC=$lc $(echo "$r" | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "Gsym/s", d["plan"])
except Exception as e: print("fail", e)')"
done; done
