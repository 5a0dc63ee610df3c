# parity tests (strict + fast + dist) and one fast bench line
timeout 600 python -m pytest tests/test_gpu_strict.py tests/test_gpu_fast.py tests/test_gpu_dist.py -x -q 2>&1 | tail -1
timeout 120 python bench.py --mode fast --steps 10 --warmup 3 --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['phase_ms'], d['ms_per_step'])"
