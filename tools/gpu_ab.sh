# A/B of apply variants: fast-path parity tests under each, then bench phases
for v in ${VARIANTS:-3}; do
  LOPT_APPLY_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_fast.py tests/test_gpu_fullsize.py tests/test_gpu_velo.py -x -q 2>&1 | tail -2
done
for v in ${BENCH_VARIANTS:-1 3}; do
  for k in 1 2; do LOPT_APPLY_VARIANT=$v timeout 300 python bench.py --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $v', round(d['ms_per_step'],4), d['roofline'].get('phase_ms'))"; done
done
