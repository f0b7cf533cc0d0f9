cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/r2m.log; : > $L
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "batched_fp32 or random_taps_all_cluster or tap_count_mask or empty_and_mixed or host_pipeline or criterion6 or device_receiver" 2>&1 | tail -2 >> $L
for env in "X=1" "DDB_NO_TMA=1"; do for cfg in cfg3 cfg3det cfg1 cfg2 cfg4; do
  env $env python bench.py --config $cfg --steps 10 --no-e2e --no-cpu --no-frontend --no-latency --no-dropin 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', '$cfg', round(d['value']/1e9,3))" >> $L
done; done
cat $L
