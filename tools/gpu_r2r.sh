#!/bin/bash
# Plan sweep for the Doppler-heavy configs (cfg3rand / cfg3det): kernel family and cluster size
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/r2r.log; : > $L
run() { # label env... -- cfg
  local lab=$1; shift
  for cfg in cfg3rand cfg3det; do
    env "$@" timeout 300 python bench.py --config $cfg --steps 5 --no-e2e --no-cpu --no-frontend --no-dropin --no-latency --no-geometry 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab', '$cfg', round(d['value']/1e9,3), {k:d['plan'].get(k) for k in ('kernel','cluster','halo_rows','threads')})" >> $L 2>&1
  done
}
run base X=1
run row DDB_KERNEL=row
run global DDB_KERNEL=global
run c4 DDB_PLAN_C=4
run c8 DDB_PLAN_C=8
run c16 DDB_PLAN_C=16
run row_c4 DDB_KERNEL=row DDB_PLAN_C=4
cat $L
