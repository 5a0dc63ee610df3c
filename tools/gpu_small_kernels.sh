timeout 900 python -m pytest tests/test_gpu_strict.py tests/test_gpu_fast.py -x -q 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sk.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_sk.csv 2>/dev/null
