#!/bin/bash
# A/B of library variants: tools/ab.sh <variant>... (libddb_<variant>.so built by build.py --variant)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/ab_${TAG:-x}.log; : > $L
for v in base "$@"; do
  if [ "$v" = base ]; then export DDB_LIB=; else export DDB_LIB=paper_2604_02266_b200/libddb_$v.so; fi
  if [ "$v" != base ]; then timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "batched_fp32_parity and tmem or random_taps_all_cluster and fp32 or tap_count_mask and tmem" 2>&1 | tail -1 | sed "s/^/$v parity: /" >> $L; fi
  for cfg in ${CFGS:-cfg3 cfg3det cfg1 cfg2}; do
    for rep in 1 2; do
    python bench.py --config $cfg --steps 10 --no-e2e --no-cpu --no-frontend --no-latency --no-dropin 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$cfg', round(d['value']/1e9,3))" >> $L
    done
  done
done
cat $L
