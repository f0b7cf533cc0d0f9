#!/bin/bash
# Evidence after the lean kernel's per-phase fold warp: GPU suite, headline bench line, cfg4 line,
# launch list, ncu --set full of the cfg3 lean kernel, phase profile
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=r2g2; L=gpurun_out/${T}.log; : > $L
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> $L
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2>gpurun_out/${T}_bench.err
for c in cfg4 cfg1 cfg2 paper128; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu --no-frontend --no-dropin > gpurun_out/${T}_bench_$c.json 2>/dev/null
done
timeout 300 python tools/phase_profile.py > gpurun_out/${T}_phase.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-latency --no-dropin > gpurun_out/${T}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sscga -s 6 -c 1 \
  -o gpurun_out/${T}_full_cfg3 -f python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu --no-latency --no-frontend --no-dropin --no-geometry > gpurun_out/${T}_ncu_cfg3.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}_full_cfg3.ncu-rep gpurun_out/${T}_ncu_cfg3.json --frames 4096 > /dev/null 2>&1
python tools/ncu_lines.py gpurun_out/${T}_full_cfg3.ncu-rep > gpurun_out/${T}_ncu_lines_cfg3.txt 2>&1
python tools/ncu_functions.py gpurun_out/${T}_full_cfg3.ncu-rep 4096 > gpurun_out/${T}_ncu_functions_cfg3.txt 2>&1
rm -f gpurun_out/${T}_full_cfg3.ncu-rep
for f in gpurun_out/${T}_bench*.json; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['value']/1e9,3), round(d['roofline']['frac'],4))" >> $L 2>&1; done
cat $L
