cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/r2k.log; : > $L
for ds in 0.0 0.1 0.2 0.4 0.6 1.0; do
  python bench.py --delay-scale $ds --steps 10 --no-e2e --no-cpu --no-frontend --no-latency --no-dropin 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ds=$ds', round(d['value']/1e9,2))" >> $L
done
cat $L
