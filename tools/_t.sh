cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in cfg3det cfg4 cfg3rand; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sscga -s 7 -c 1 \
    -o gpurun_out/r2x_full_${c} -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --no-latency --no-frontend --no-dropin --no-geometry > gpurun_out/r2x_ncu_${c}.log 2>&1
done
ls -la gpurun_out/r2x_full_*
