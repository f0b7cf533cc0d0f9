#!/bin/bash
# TMEM-kernel plan sweep on cfg3: cluster size x warps per lane quarter x smem cap (CTAs per SM).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
run() {
  r=$(env "$@" timeout 120 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-latency ${BENCH_ARGS} 2>/dev/null | tail -1)
  echo "$* :: $(echo "$r" | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "Gsym/s", d["plan"])
except Exception as e: print("fail", e)')"
}
run DDB_PLAN_C=2
run DDB_PLAN_C=4 DDB_PLAN_WQ=4
run DDB_PLAN_C=4 DDB_PLAN_WQ=2
run DDB_PLAN_C=4 DDB_PLAN_WQ=2 DDB_PLAN_SMEM_CAP=112000
run DDB_PLAN_C=8 DDB_PLAN_WQ=4 DDB_PLAN_SMEM_CAP=112000
run DDB_PLAN_C=8 DDB_PLAN_WQ=2 DDB_PLAN_SMEM_CAP=112000
run DDB_PLAN_C=8 DDB_PLAN_WQ=1 DDB_PLAN_SMEM_CAP=55000
run DDB_PLAN_C=8 DDB_PLAN_WQ=1 DDB_PLAN_SMEM_CAP=74000
run DDB_KERNEL=row
