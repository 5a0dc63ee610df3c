timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_velo.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -x -q 2>&1 | tail -2
for k in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('phase_ms'))"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s5.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_s5.csv 2>/dev/null | grep stats
