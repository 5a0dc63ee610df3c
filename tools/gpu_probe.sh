set -x
python tools/probe_umma.py
export LOPT_BENCH_MODE=fast
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^(apply|factor|prep|stats)" --csv --log-file gpurun_out/launches_fast3.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:apply_tc -s 3 -c 1 -o gpurun_out/prof_apply3 $B > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:factor_partials -s 3 -c 1 -o gpurun_out/prof_factor3 $B > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stats_fast -s 3 -c 1 -o gpurun_out/prof_stats3 $B > /dev/null 2>&1
ls gpurun_out
