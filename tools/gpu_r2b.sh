#!/bin/bash
# Round-2 GPU pass B: residency probe, new parity / harness / reference-suite tests,
# the whole -m gpu suite, smoke and one bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-r2b}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${T}_smi.txt 2>&1
nproc >> gpurun_out/${T}_smi.txt; lscpu | grep "Model name" >> gpurun_out/${T}_smi.txt
(cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O2 resident.cu -o resident && timeout 120 ./resident) > gpurun_out/${T}_resident.txt 2>&1
timeout 1500 python -m pytest -q tests/test_sweep_parity.py tests/test_harness_gpu.py tests/test_reference_suite.py \
  "tests/test_gpu_parity.py::test_fused_epilogue_labels_and_llr_magnitudes" -rA > gpurun_out/${T}_new_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_new_tests.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 600 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${T}_bench.log
tail -3 gpurun_out/${T}_new_tests.log gpurun_out/${T}_pytest_gpu.log gpurun_out/${T}_smoke.log gpurun_out/${T}_bench.log
