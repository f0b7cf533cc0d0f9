timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/ps_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/ps_pytest.log; grep FAIL gpurun_out/ps_pytest.log | head -5
timeout 300 python tools/receiver_breakdown.py > gpurun_out/ps_rb.log 2>&1; head -8 gpurun_out/ps_rb.log
timeout 600 python bench.py --config paper --no-cpu > gpurun_out/ps_paper.log 2>&1; grep '^{' gpurun_out/ps_paper.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); L=d['latency']; print(d['value']/1e9, {k: (round(v,4) if isinstance(v,float) else v) for k,v in L.items() if k!='what'})"
