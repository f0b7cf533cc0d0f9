cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-r2n}
timeout 900 python -m pytest -q tests/test_multirank_gpu.py -rA > gpurun_out/${T}_multirank.log 2>&1; echo rc=$? >> gpurun_out/${T}_multirank.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo rc=$? >> gpurun_out/${T}_bench.log
timeout 300 python bench.py --config cfg3rand --no-e2e --no-cpu --no-frontend --no-latency --no-dropin > gpurun_out/${T}_bench_cfg3rand.log 2>&1
tail -3 gpurun_out/${T}_multirank.log
python - <<'PY'
import json
d=json.loads([l for l in open('gpurun_out/r2n_bench.log') if l.startswith('{')][-1])
print(d['value']/1e9, d['roofline']['frac'], d['tap_geometry'], d['cpu_baseline'], d['e2e']['value']/1e9, d['dropin'])
d=json.loads([l for l in open('gpurun_out/r2n_bench_cfg3rand.log') if l.startswith('{')][-1])
print('cfg3rand', d['value']/1e9, d['roofline']['frac'])
PY
