for d in 0 8192 32768 131072 0; do
echo "dbg=$d"; LOPT_APPLY_DEBUG=$d timeout 300 python bench.py --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('phase_ms'))"
done
