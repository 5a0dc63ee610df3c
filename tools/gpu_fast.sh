set -x
timeout 300 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_fast.py -x -q 2>&1 | tail -25
LOPT_BENCH_MODE=fast timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -3
