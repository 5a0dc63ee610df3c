set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1.json
timeout 300 python bench.py --mode strict --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/bench_r1_strict.json
timeout 600 python bench.py --workload gpt2_medium --feature-set velo --no-cpu --no-e2e --no-velo --steps 10 2>&1 | tail -1 > gpurun_out/bench_r1_gpt2_velo.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_r1_reference.json
cut -c1-300 gpurun_out/bench_r1_gpt2_velo.json gpurun_out/bench_r1_reference.json
