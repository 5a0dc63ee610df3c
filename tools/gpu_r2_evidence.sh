# Round-2 evidence: smoke, full GPU parity suite, default bench line, launch list, ncu --set full of the streaming kernels
set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r2.json
cut -c1-3000 gpurun_out/bench_r2.json
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"factor_partials|stats_fast_kernel|apply_[a-z]+_kernel" -s 9 -c 3 -o gpurun_out/prof_r2_final $B > /dev/null 2>&1
ls gpurun_out | tail -5
