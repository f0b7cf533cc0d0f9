#!/bin/bash
# cfg4 evidence after the frame-sized ghost pushes: bench line, ncu --set full of the general kernel, per-line view
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=r2v
timeout 600 python bench.py --config cfg4 --no-e2e --no-cpu --no-frontend --no-dropin > gpurun_out/${T}_bench_cfg4.json 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sscga -s 7 -c 1 \
  -o gpurun_out/${T}_full_cfg4 -f python bench.py --config cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-latency --no-frontend --no-dropin --no-geometry > gpurun_out/${T}_ncu_cfg4.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}_full_cfg4.ncu-rep gpurun_out/${T}_ncu_cfg4.json --frames 1024 > /dev/null 2>&1
python tools/ncu_lines.py gpurun_out/${T}_full_cfg4.ncu-rep > gpurun_out/${T}_ncu_lines_cfg4.txt 2>&1
rm -f gpurun_out/${T}_full_cfg4.ncu-rep
tail -c 400 gpurun_out/${T}_bench_cfg4.json
