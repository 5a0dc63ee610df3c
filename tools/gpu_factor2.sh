timeout 900 python -m pytest tests/test_gpu_strict.py tests/test_gpu_fast.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
for t in 131072 65536 262144; do
echo "tile=$t"; LOPT_FACTOR_TILE=$t timeout 300 python bench.py --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('phase_ms'))"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f2.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_f2.csv | head -3
