#!/bin/bash
# L2-mirror route A/B: GPU suite, then the Doppler configs with / without the mirror and its |d_l| threshold
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/r2s.log; : > $L
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 >> $L
run() { local lab=$1; shift
  for cfg in ${CFGS:-cfg3rand cfg3det cfg4 cfg3}; do
    env "$@" timeout 300 python bench.py --config $cfg --steps 10 --no-e2e --no-cpu --no-frontend --no-dropin --no-latency --no-geometry 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lab', '$cfg', round(d['value']/1e9,3))" >> $L 2>&1
  done
}
run mirror X=1
run nomirror DDB_NO_MIRROR=1
run mirror_dl1 DDB_MIRROR_DL=1
run mirror X=1
cat $L
