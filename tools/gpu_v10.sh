timeout 400 python -m pytest tests/test_gpu_fast.py tests/test_gpu_velo.py -x -q 2>&1 | tail -2
for d in 0 31; do
  echo "dbg=$d"; LOPT_APPLY_DEBUG=$d timeout 120 python bench.py --mode fast --steps 10 --warmup 3 --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['phase_ms'])"
done
bash tools/gpu_prof.sh v10
