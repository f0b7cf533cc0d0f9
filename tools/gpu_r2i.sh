cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-r2i}
python tools/dropin_timing.py > gpurun_out/${T}_dropin.json 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
cat gpurun_out/${T}_dropin.json; tail -4 gpurun_out/${T}_pytest_gpu.log; grep -n "criterion 10" gpurun_out/reference_suite_fp64.log
