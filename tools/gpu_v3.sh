set -x
timeout 600 python -m pytest tests/test_gpu_fast.py tests/test_gpu_dist.py -x -q -s 2>&1 | grep -E "relL2|elementwise|passed|failed|Error|assert" | head -30
LOPT_BENCH_MODE=fast timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-900
