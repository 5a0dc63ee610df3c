for t in 131072 114688 98304 73728 131072; do
echo "tile=$t"; LOPT_FACTOR_TILE=$t timeout 300 python bench.py --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('phase_ms'))"
done
