timeout 900 python -m pytest tests -m gpu -q > gpurun_out/dt_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/dt_pytest.log; grep FAIL gpurun_out/dt_pytest.log | head
