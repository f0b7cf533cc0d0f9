timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/op2_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/op2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/op2_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/op2_bench.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/op2_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']/1e9,3), round(d['roofline']['frac'],4), round(d['e2e']['value']/1e9,3), d['e2e']['pcie']['frac'], d['cpu_baseline']['value']/1e6, d['latency']['p50_ms'], d['latency']['receiver_p999_ms'], d['clocks'])"
timeout 300 python tools/phase_profile.py > gpurun_out/op2_phase.log 2>&1
for c in cfg3det paper128 cfg2; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/op2_$c.log 2>&1; grep '^{' gpurun_out/op2_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$c', round(d['value']/1e9,3))"; done
