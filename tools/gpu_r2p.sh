cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/r2p.log; : > $L
timeout 1500 python -m pytest -q -x tests/test_gpu_parity.py tests/test_sweep_parity.py tests/test_harness_gpu.py 2>&1 | tail -3 >> $L
CFGS="cfg3 cfg3det cfg3rand cfg1 cfg2 cfg4" TAG=split bash tools/ab.sh head >> $L 2>&1
cat $L
