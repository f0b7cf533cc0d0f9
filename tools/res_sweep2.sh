#!/bin/bash
# Residency sweep on the small grids and cfg4 (measured 2+ TMEM CTAs per SM).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-r2d}
L=gpurun_out/${T}_sweep.log
run() {  # name cfg env...
  local name=$1 cfg=$2; shift 2
  echo "=== $name $cfg $*" >> $L
  env "$@" timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu --no-latency --no-frontend > gpurun_out/${T}_${name}_${cfg}.json 2>>$L
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], round(d['value']/1e9,2), 'Gsym/s', round(d['roofline']['frac'],3), d.get('plan'))" gpurun_out/${T}_${name}_${cfg}.json $name $cfg >> $L 2>&1
}
env timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "batched_fp32_parity and tmem or random_taps_all_cluster and fp32 or tap_count_mask and tmem" >> $L 2>&1
run def cfg1 X=1
run one cfg1 DDB_TM_CTAS_PER_SM=1
run w1 cfg1 DDB_PLAN_WQ=1
run w1s cfg1 DDB_PLAN_WQ=1 DDB_PLAN_SMEM_CAP=40000
run def cfg2 X=1
run w2 cfg2 DDB_PLAN_WQ=2 DDB_PLAN_SMEM_CAP=112000
run w1 cfg2 DDB_PLAN_WQ=1 DDB_PLAN_SMEM_CAP=56000
run def paper128 X=1
run w2 paper128 DDB_PLAN_WQ=2 DDB_PLAN_SMEM_CAP=112000
run def cfg4 X=1
run c16 cfg4 DDB_PLAN_C=16 DDB_PLAN_WQ=2 DDB_PLAN_SMEM_CAP=112000
grep -i "gsym\|passed\|failed\|error" $L
