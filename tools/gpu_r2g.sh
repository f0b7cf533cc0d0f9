cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python tools/dropin_timing.py > gpurun_out/r2g_dropin.json 2>&1
(cd tools/ubench && for m in 0 1 2; do for t in synccheck racecheck memcheck; do echo "== $t mode $m"; compute-sanitizer --tool $t ./san_tmem $m 2>&1 | grep -v "^=========     \|Host Frame" | head -8; done; done) > gpurun_out/r2g_san_tmem.txt 2>&1
timeout 900 python -m pytest -q tests/test_reference_suite.py tests/test_gpu_parity.py -k "reference_suite or detect_paths" > gpurun_out/r2g_tests.log 2>&1; echo rc=$? >> gpurun_out/r2g_tests.log
cat gpurun_out/r2g_dropin.json gpurun_out/r2g_san_tmem.txt; tail -3 gpurun_out/r2g_tests.log; grep -n "criterion 10" gpurun_out/reference_suite_fp64.log
