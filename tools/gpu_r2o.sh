cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/r2o.log; : > $L
timeout 900 python -m pytest -q tests/test_gpu_parity.py -k "random or batched_fp32 or tap_count or empty_and_mixed or criterion or detect or sweep" 2>&1 | tail -3 >> $L
for cfg in cfg3rand cfg3 cfg3det cfg4 cfg1 cfg2; do
  python bench.py --config $cfg --steps 10 --no-e2e --no-cpu --no-frontend --no-latency --no-dropin --no-geometry 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value']/1e9,3), round(d['roofline']['frac'],4))" >> $L
done
cat $L
