timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/dn_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/dn_pytest.log
