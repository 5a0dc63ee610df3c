# bench apply phase under LOPT_APPLY_DEBUG switch values ($DBGS), two runs each
for d in ${DBGS:-0 1 2 3}; do
  for k in 1 2; do LOPT_APPLY_DEBUG=$d timeout 300 python bench.py --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg $d', round(d['ms_per_step'],4), d['roofline'].get('phase_ms'))"; done
done
