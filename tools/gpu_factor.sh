B="python bench.py --mode fast --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:factor_partials -s 3 -c 1 -o gpurun_out/prof_factor_$1 $B > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv $B > /dev/null 2>&1
