timeout 900 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -3
for st in range owner; do
LOPT_DIST_BACKEND=gloo LOPT_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu --no-e2e --strategy $st 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['ms_per_step_without_param_exchange'], d['config']['parallelism'], d['roofline']['phase_ms'], d['velo']['ms_per_step'])"
done
