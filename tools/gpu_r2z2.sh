#!/bin/bash
# Row-block tap exchange (cfg3 lean frames): GPU suite, A/B against the previous HEAD, phase profile
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/r2z2.log; : > $L
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> $L
CFGS="cfg3 cfg3det paper128 cfg2" TAG=r2z2 bash tools/ab.sh head >> $L 2>&1
CFGS="cfg3" TAG=r2z3 bash tools/ab.sh head >> $L 2>&1
timeout 300 python tools/phase_profile.py > gpurun_out/r2z2_phase.json 2>&1
cat $L
