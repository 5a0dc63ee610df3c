timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_dist.py tests/test_gpu_velo.py -x -q 2>&1 | tail -2
for t in 131072 65536 32768 16384; do
echo "tile=$t"; LOPT_FACTOR_TILE=$t timeout 300 python bench.py --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('phase_ms'))"
done
