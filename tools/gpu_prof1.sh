set -x
timeout 600 python -m pytest tests/test_gpu_fast.py -x -q 2>&1 | tail -8
LOPT_BENCH_MODE=fast timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_fast.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo > /dev/null 2>&1
tail -45 gpurun_out/launches_fast.csv | cut -c1-250
