for d in 0 4 16 8 28 30 31; do
  echo -n "dbg=$d "; LOPT_APPLY_DEBUG=$d timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['phase_ms']['apply'],3))"
done
