export DDB_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-latency --no-frontend > gpurun_out/mr_bench.log 2>&1; echo "torchrun rc=$?"
grep -c '^{' gpurun_out/mr_bench.log; grep '^{' gpurun_out/mr_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['n_gpus'], d['value']/1e9, d['e2e']['value']/1e9 if d['e2e'] else None, d['scaling'], d['gpu_launches'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 --cpu-seconds 2 > gpurun_out/mr_ref.log 2>&1; echo "ref rc=$?"; grep -c '^{' gpurun_out/mr_ref.log
tail -3 gpurun_out/mr_bench.log
