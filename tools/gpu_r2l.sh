cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/r2l.log; : > $L
for ds in 0.1 0.3; do
for cfgv in "DDB_PLAN_C=2" "DDB_PLAN_C=4 DDB_PLAN_WQ=2 DDB_PLAN_SMEM_CAP=112000" "DDB_PLAN_C=4 DDB_PLAN_WQ=2 DDB_PLAN_SMEM_CAP=112000 DDB_TM_CTAS_PER_SM=1" "DDB_PLAN_C=8 DDB_PLAN_WQ=1 DDB_PLAN_SMEM_CAP=56000"; do
  env $cfgv python bench.py --delay-scale $ds --steps 10 --no-e2e --no-cpu --no-frontend --no-latency --no-dropin 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ds=$ds', '$cfgv', round(d['value']/1e9,2), d['plan']['ctas_per_sm'], d['ber'])" >> $L
done; done
cat $L
