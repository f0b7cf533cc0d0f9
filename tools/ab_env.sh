#!/bin/bash
# A/B of environment settings on one library: tools/ab_env.sh "ENV=.." "ENV=.." ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/abenv_${TAG:-x}.log; : > $L
for v in "$@"; do
  for cfg in ${CFGS:-cfg3 cfg3det cfg1 cfg2}; do
    for rep in 1 2; do
    env $v python bench.py --config $cfg --steps 10 --no-e2e --no-cpu --no-frontend --no-latency --no-dropin --no-geometry 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$cfg', round(d['value']/1e9,3))" >> $L
    done
  done
done
cat $L
