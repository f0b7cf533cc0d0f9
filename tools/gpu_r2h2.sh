#!/bin/bash
# Final HEAD check: GPU suite, smoke, headline bench line, cfg4 / cfg1 / cfg2 / paper128 lines, launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=r2h2; L=gpurun_out/${T}.log; : > $L
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -1 >> $L
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2>gpurun_out/${T}_bench.err
for c in cfg4 cfg1 cfg2 paper128 cfg3det cfg3rand; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu --no-frontend --no-dropin > gpurun_out/${T}_bench_$c.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-latency --no-dropin > gpurun_out/${T}_ncu_bench.log 2>&1
for f in gpurun_out/${T}_bench*.json; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['value']/1e9,3), round(d['roofline']['frac'],4))" >> $L 2>&1; done
cat $L
