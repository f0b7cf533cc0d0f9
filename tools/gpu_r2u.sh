#!/bin/bash
# A/B: first-tap accumulator init (base) vs zeroed (noinit) vs HEAD; ghost pushes sized to the frame's |d_l|
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/r2u.log; : > $L
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> $L
CFGS="cfg3 cfg4 cfg2 cfg1 cfg3det" TAG=r2u bash tools/ab.sh noinit head >> $L 2>&1
CFGS="cfg3 cfg4" TAG=r2u2 bash tools/ab.sh head >> $L 2>&1
cat $L
