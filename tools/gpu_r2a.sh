#!/bin/bash
# Round-2 GPU pass A: residency probe, new parity / harness / reference-suite tests,
# compute-sanitizer on every fused kernel, then the whole -m gpu suite.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-r2a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${T}_smi.txt 2>&1
nproc >> gpurun_out/${T}_smi.txt
(cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O2 resident.cu -o resident && timeout 120 ./resident) > gpurun_out/${T}_resident.txt 2>&1
timeout 2400 python -m pytest -x -q tests/test_sweep_parity.py tests/test_harness_gpu.py tests/test_reference_suite.py \
  "tests/test_gpu_parity.py::test_fused_epilogue_labels_and_llr_magnitudes" -rA > gpurun_out/${T}_new_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_new_tests.log
SAN=gpurun_out/${T}_sanitizer.log
: > $SAN
for tool in memcheck racecheck synccheck; do
  for args in "--kernel tmem --grid cfg1 --batch 4" "--kernel tmem --grid cfg3 --batch 2" "--kernel tmem --grid cfg3 --batch 2 --doppler" \
              "--kernel row --grid cfg1 --batch 4" "--kernel row --grid cfg3 --batch 2 --precision fp64" \
              "--kernel global --grid cfg1 --batch 2" "--kernel global --grid cfg1 --batch 12" "--kernel tmem --grid cfg4 --batch 1 --doppler"; do
    echo "=== $tool $args" >> $SAN
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $args >> $SAN 2>&1
    echo "rc=$?" >> $SAN
  done
done
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
tail -3 gpurun_out/${T}_new_tests.log gpurun_out/${T}_pytest_gpu.log; grep -c "ERROR SUMMARY: 0" $SAN; grep "ERROR SUMMARY" $SAN | sort | uniq -c
