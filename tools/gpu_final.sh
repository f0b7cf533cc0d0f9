#!/bin/bash
# Final evidence pass: full bench line (headline), every config, fp64 line, strong scaling,
# the reference arm, the ncu launch list of the bench command and one --set full capture per config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-r2f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2>gpurun_out/${T}_bench.err
for c in cfg1 cfg2 cfg4 cfg3det cfg3rand paper paper128; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu --no-frontend --no-dropin > gpurun_out/${T}_bench_$c.json 2>/dev/null
done
timeout 300 python bench.py --precision fp64 --no-e2e --no-cpu --no-frontend --no-latency --no-geometry > gpurun_out/${T}_bench_fp64.json 2>/dev/null
timeout 600 python bench.py --impl reference > gpurun_out/${T}_reference.json 2>/dev/null
timeout 300 python tools/phase_profile.py > gpurun_out/${T}_phase.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-latency --no-dropin > gpurun_out/${T}_ncu_bench.log 2>&1
# one --set full capture per config: the lean kernel for cfg3 / cfg1 (-s 6: after the
# 3 warm-up solves of 2 launches each), the general one for cfg3det / cfg4 / cfg3rand (-s 7);
# summarised here and the reports removed (gpurun_out travels back only under 64 MiB)
for cs in "cfg3 6 4096" "cfg1 6 4096" "cfg2 6 1024" "cfg3det 7 4096" "cfg4 7 1024" "cfg3rand 7 4096"; do
  set -- $cs
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sscga -s $2 -c 1 \
    -o gpurun_out/${T}_full_$1 -f python bench.py --config $1 --steps 1 --warmup 3 --no-e2e --no-cpu --no-latency --no-frontend --no-dropin --no-geometry > gpurun_out/${T}_ncu_$1.log 2>&1
  python tools/ncu_summary.py gpurun_out/${T}_full_$1.ncu-rep gpurun_out/${T}_ncu_$1.json --frames $3 > /dev/null 2>&1
  python tools/ncu_lines.py gpurun_out/${T}_full_$1.ncu-rep > gpurun_out/${T}_ncu_lines_$1.txt 2>&1
  python tools/ncu_functions.py gpurun_out/${T}_full_$1.ncu-rep $3 > gpurun_out/${T}_ncu_functions_$1.txt 2>&1
  rm -f gpurun_out/${T}_full_$1.ncu-rep
done
ls gpurun_out/${T}_*
