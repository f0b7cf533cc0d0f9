timeout 900 python -m pytest tests -m gpu -x -q -k "Synthesis or receive or criterion6" > gpurun_out/syn_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/syn_pytest.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-e2e --no-latency > gpurun_out/syn_bench$i.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/syn_bench$i.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); f=d['frontend']; print(d['value']/1e9, {k: f[k] for k in f if k != 'what'})"
done
