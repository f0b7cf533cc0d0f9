#!/bin/bash
# Residency sweep: the cfg3 (and cfg3det) fused solve at 1, 2 and 4 CTAs per SM
# (cluster 2 / 4 / 8, 512 / 256 / 128 threads), parity subset first.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-r2c}
run() {  # name env...
  local name=$1; shift
  echo "=== $name $*" >> gpurun_out/${T}_sweep.log
  env "$@" timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "batched_fp32_parity and tmem or random_taps_all_cluster and fp32 or tap_count_mask and tmem" >> gpurun_out/${T}_sweep.log 2>&1
  for cfg in cfg3 cfg3det; do
    env "$@" timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu --no-latency --no-frontend > gpurun_out/${T}_${name}_${cfg}.json 2>>gpurun_out/${T}_sweep.log
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], round(d['value']/1e9,2), 'Gsym/s', round(d['roofline']['frac'],3), d.get('plan'))" gpurun_out/${T}_${name}_${cfg}.json $name $cfg >> gpurun_out/${T}_sweep.log 2>&1
  done
}
run c2 DDB_PLAN_C=2
run c4w2 DDB_PLAN_C=4 DDB_PLAN_WQ=2 DDB_PLAN_SMEM_CAP=112000
run c8w1 DDB_PLAN_C=8 DDB_PLAN_WQ=1 DDB_PLAN_SMEM_CAP=56000
run c4w2_1 DDB_PLAN_C=4 DDB_PLAN_WQ=2 DDB_PLAN_SMEM_CAP=112000 DDB_TM_CTAS_PER_SM=1
grep -v "^\.\|^$" gpurun_out/${T}_sweep.log | grep -i "gsym\|passed\|failed\|error" 
