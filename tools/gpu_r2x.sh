#!/bin/bash
# Doppler-tap coefficient tables (two-CTA plans): GPU suite, then A/B against the previous HEAD
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/r2x.log; : > $L
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "doppler_coefficient_tables or ghost" 2>&1 | tail -2 >> $L
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> $L
CFGS="cfg3det cfg3 cfg3rand cfg2 cfg1 cfg4" TAG=r2x bash tools/ab.sh head >> $L 2>&1
cat $L
