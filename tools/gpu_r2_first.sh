# Round-2 first look: smoke, A/B of the apply variants (1 = role-specialized, 2 = unified warpgroups), GPU suite
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for v in 1 2; do
  for k in 1 2; do LOPT_APPLY_VARIANT=$v timeout 300 python bench.py --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $v', d['ms_per_step'], d['roofline'].get('phase_ms'))"; done
done
LOPT_APPLY_VARIANT=2 timeout 300 python -m pytest tests/test_gpu_fast.py -x -q 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8
