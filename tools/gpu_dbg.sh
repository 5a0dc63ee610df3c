for d in 0 31; do
  echo "dbg=$d"; LOPT_APPLY_DEBUG=$d timeout 300 python bench.py --mode fast --steps 10 --warmup 3 --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['phase_ms']['apply'])"
done
timeout 300 python -m pytest tests/test_gpu_fast.py -x -q 2>&1 | tail -2
