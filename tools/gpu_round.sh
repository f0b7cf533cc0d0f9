#!/bin/bash
# One GPU-box pass: parity suite, smoke, bench, phase profile, ncu launch list + full capture.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-cur}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
timeout 300 python tools/phase_profile.py > gpurun_out/${TAG}_phase.log 2>&1
if [ -z "$SKIP_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-latency > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sscga -s 3 -c 1 \
  -o gpurun_out/${TAG}_full -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-latency > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
for f in gpurun_out/${TAG}_*.log; do tail -n 3 "$f"; done
