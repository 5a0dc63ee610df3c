# Round evidence: smoke, full GPU parity suite, bench lines (fast default, strict), launch list, ncu full of the three streaming kernels
set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1.json
cut -c1-4000 gpurun_out/bench_r1.json
timeout 300 python bench.py --mode strict --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/bench_r1_strict.json
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"factor_partials|stats_fast_kernel|apply_tc" -s 9 -c 3 -o gpurun_out/prof_r1_final $B > /dev/null 2>&1
ls gpurun_out | tail -5
