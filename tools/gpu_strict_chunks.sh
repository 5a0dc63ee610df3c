for c in 8192,4096 8192,16384 32768,16384 32768,65536; do
echo "chunks=$c"; LOPT_STRICT_CHUNKS=$c timeout 300 python bench.py --mode strict --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('phase_ms'))"
done
