#!/bin/bash
# ncu --set full of the general kernel on cfg3rand (with and without the L2 mirror), per-line stalls
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for v in mir nomir; do
  if [ $v = nomir ]; then export DDB_NO_MIRROR=1; fi
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sscga -s 7 -c 1 \
    -o gpurun_out/r2t_$v -f python bench.py --config cfg3rand --steps 1 --warmup 3 --no-e2e --no-cpu --no-latency --no-frontend --no-dropin --no-geometry > gpurun_out/r2t_ncu_$v.log 2>&1
  python tools/ncu_summary.py gpurun_out/r2t_$v.ncu-rep gpurun_out/r2t_ncu_$v.json --frames 4096 > /dev/null 2>&1
  python tools/ncu_lines.py gpurun_out/r2t_$v.ncu-rep > gpurun_out/r2t_lines_$v.txt 2>&1
  rm -f gpurun_out/r2t_$v.ncu-rep
done
ls gpurun_out/r2t*
