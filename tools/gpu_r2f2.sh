#!/bin/bash
# A/B: the CTA-partials fold by the lightest row block of the next MVM (DDB_FOLD_SPLIT=1) vs a middle one
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/r2f2.log; : > $L
CFGS="cfg3 cfg3det paper128 cfg4" TAG=r2f2 bash tools/ab.sh fold >> $L 2>&1
CFGS="cfg3" TAG=r2f3 bash tools/ab.sh fold >> $L 2>&1
cat $L
