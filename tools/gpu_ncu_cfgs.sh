#!/bin/bash
# ncu --set full captures of the fused solve for every config (one launch each)
# plus the phase profile of cfg3; sanitizer pass on the fused kernels at small batches.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-r2e}
for cfg in cfg3 cfg1 cfg2 cfg4 cfg3det; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sscga -s 3 -c 1 \
    -o gpurun_out/${T}_full_${cfg} -f python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu --no-latency --no-frontend > gpurun_out/${T}_ncu_${cfg}.log 2>&1
  echo "$cfg rc=$?" >> gpurun_out/${T}_ncu_status.txt
done
timeout 300 python tools/phase_profile.py > gpurun_out/${T}_phase.log 2>&1
SAN=gpurun_out/${T}_sanitizer.log
: > $SAN
for tool in memcheck racecheck synccheck; do
  for args in "--kernel tmem --grid cfg1 --batch 4" "--kernel tmem --grid cfg3 --batch 2" "--kernel tmem --grid cfg3 --batch 2 --doppler" \
              "--kernel row --grid cfg3 --batch 2 --precision fp64" "--kernel global --grid cfg1 --batch 2" "--kernel global --grid cfg1 --batch 12"; do
    echo "=== $tool $args" >> $SAN
    timeout 300 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $args >> $SAN 2>&1
    echo "rc=$?" >> $SAN
  done
done
cat gpurun_out/${T}_ncu_status.txt; grep "ERROR SUMMARY\|^===\|^rc=" $SAN
