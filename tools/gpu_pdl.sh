# programmatic dependent launch on the fast-path chain vs LOPT_NO_PDL=1 (same box)
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do for v in 0 1; do
  LOPT_NO_PDL=$v timeout 300 python bench.py --steps 30 --warmup 10 --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no_pdl=$v', round(d['ms_per_step'],4), d['step_ms_p10_p50_p90'], {k: round(x,4) for k,x in d['roofline']['phase_ms'].items()})"
done; done
for v in 0 1; do
  LOPT_NO_PDL=$v timeout 300 python bench.py --workload gpt2_medium --feature-set velo --steps 10 --warmup 5 --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gpt2 no_pdl=$v', round(d['ms_per_step'],4), d['step_ms_p10_p50_p90'])"
done
