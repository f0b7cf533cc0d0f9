#!/bin/bash
# Re-entry check of HEAD: the whole -m gpu suite, smoke, and the headline bench line + configs
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/r2q.log; : > $L
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 >> $L
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1
timeout 900 python bench.py > gpurun_out/r2q_bench.json 2>gpurun_out/r2q_bench.err
for c in cfg3det cfg4 cfg3rand cfg1; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu --no-frontend --no-dropin --no-latency --no-geometry 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']/1e9,3), round(d['roofline']['frac'],4))" >> $L
done
cat $L
