cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-r2h}
python tools/dropin_timing.py > gpurun_out/${T}_dropin.json 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python bench.py --no-e2e --no-cpu --no-frontend --no-latency > gpurun_out/${T}_bench.log 2>&1
cat gpurun_out/${T}_dropin.json; tail -4 gpurun_out/${T}_pytest_gpu.log; grep -n "criterion 10" gpurun_out/reference_suite_fp64.log
python -c "import json; d=json.loads(open('gpurun_out/${T}_bench.log').read().strip().splitlines()[-1]); print(d['value']/1e9, d['dropin'])"
