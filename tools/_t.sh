cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sscga -s 6 -c 1 -o gpurun_out/r2y_full_cfg3 -f python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu --no-latency --no-frontend --no-dropin --no-geometry > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sscga -s 7 -c 1 -o gpurun_out/r2y_full_cfg3det -f python bench.py --config cfg3det --steps 1 --warmup 3 --no-e2e --no-cpu --no-latency --no-frontend --no-dropin --no-geometry > /dev/null 2>&1
ls gpurun_out/r2y*
