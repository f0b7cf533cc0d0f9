#!/bin/bash
# Solve time vs taps per frame (cfg3 grid): fixed per-frame overhead and per-tap slope of each kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for k in tmem row; do for p in 1 2 4 6 12; do
  r=$(DDB_KERNEL=$k timeout 120 python bench.py --steps 5 --warmup 3 --paths $p --no-e2e --no-cpu --no-latency 2>/dev/null | tail -1)
  echo "$k P=$p $(echo "$r" | python -c 'import json,sys
d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "Gsym/s", round(d["ms_per_step"],3), "ms/step", round(d["ms_per_step"]*1e6/4096*74/1e3*1.965,1), "kcyc/frame/cluster")')"
done; done
