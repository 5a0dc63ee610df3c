set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -30
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -3 > gpurun_out/bench1.txt
cat gpurun_out/bench1.txt
