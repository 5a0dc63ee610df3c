timeout 400 python -m pytest tests/test_gpu_fast.py -x -q 2>&1 | tail -2
timeout 120 python bench.py --mode fast --steps 10 --warmup 3 --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['phase_ms'], d['ms_per_step'])"
B="python bench.py --mode fast --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stats_fast -s 3 -c 1 -o gpurun_out/prof_stats_$1 $B > /dev/null 2>&1
