# Round evidence: smoke, full GPU parity suite, default bench line, launch list, ncu of apply
set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1.json
cut -c1-3000 gpurun_out/bench_r1.json
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:apply_tc -s 3 -c 1 -o gpurun_out/prof_apply_r1 $B > /dev/null 2>&1
ls gpurun_out | tail -5
