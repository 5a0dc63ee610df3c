timeout 600 python -m pytest tests/test_gpu_fast.py -x -q -k step_host 2>&1 | tail -2
for c in 8 16 32; do
echo "chunks=$c"; LOPT_E2E_CHUNKS=$c timeout 300 python bench.py --no-cpu --no-velo --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'])"
done
