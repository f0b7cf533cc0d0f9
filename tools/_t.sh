cd "${GRAFT_REPO_ROOT:-/root/repo}"
export DDB_LIB=paper_2604_02266_b200/libddb_sr.so
for i in 1 2 3; do timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_sweep_parity.py -k "random or batched or sweep or cfg4 or criterion or device_receiver or frontend or synth" 2>&1 | tail -1; done
unset DDB_LIB
CFGS="cfg3det cfg4 cfg3rand cfg3" TAG=sr bash tools/ab.sh sr
