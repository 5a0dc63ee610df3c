# One GPU call: parity tests, benches (fast + strict), launch list.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --mode fast --steps 20 --warmup 5 2>&1 | tail -1 > gpurun_out/bench_fast.json
timeout 300 python bench.py --mode strict --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/bench_strict.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fast.csv python bench.py --mode fast --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo > /dev/null 2>&1
cut -c1-1500 gpurun_out/bench_fast.json
