timeout 300 python -m pytest tests/test_gpu_fast.py -x -q -k "steps_vs_oracle" 2>&1 | tail -1
for k in 1 2 3; do timeout 300 python bench.py --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('phase_ms'))"; done
