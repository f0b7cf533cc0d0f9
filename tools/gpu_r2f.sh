#!/bin/bash
# Round-2 pass F: whole -m gpu suite, smoke, bench (default, fp64, strong), sanitizer isolation runs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-r2f}
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${T}_bench.log
timeout 300 python bench.py --precision fp64 --no-e2e --no-cpu --no-frontend --no-latency > gpurun_out/${T}_bench_fp64.log 2>&1
timeout 300 python bench.py --scaling strong --no-e2e --no-cpu --no-frontend --no-latency --no-dropin > gpurun_out/${T}_bench_strong.log 2>&1
for c in cfg1 cfg2 paper128 cfg3det cfg4 paper; do
  timeout 300 python bench.py --config $c --no-e2e --no-cpu --no-frontend --no-latency --no-dropin > gpurun_out/${T}_bench_$c.log 2>&1
done
SAN=gpurun_out/${T}_sanitizer.log
: > $SAN
for tool in synccheck racecheck; do
  for args in "--kernel tmem --grid cfg1 --batch 4" "--kernel row --grid cfg1 --batch 4 --precision fp64"; do
    echo "=== DDB_NO_CLUSTER_ATTR=1 $tool $args" >> $SAN
    DDB_NO_CLUSTER_ATTR=1 timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $args >> $SAN 2>&1
    echo "rc=$?" >> $SAN
  done
done
tail -3 gpurun_out/${T}_pytest_gpu.log; grep "^===\|SUMMARY\|^rc" $SAN
for f in gpurun_out/${T}_bench*.log; do python - "$f" <<'PY'
import json,sys
for ln in open(sys.argv[1]):
    if ln.startswith('{'):
        d=json.loads(ln); print(sys.argv[1].split('/')[-1], round(d['value']/1e9,3), d['roofline']['bound'], round(d['roofline']['frac'],3), d.get('dropin'), d.get('plan',{}).get('ctas_per_sm'))
PY
done
