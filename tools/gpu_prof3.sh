set -x
export LOPT_BENCH_MODE=fast
B="python bench.py --mode fast --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
timeout 120 python tools/probe_umma.py > gpurun_out/probe.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:apply_tc -s 3 -c 1 -o gpurun_out/prof_apply_v4 $B > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stats_fast -s 3 -c 1 -o gpurun_out/prof_stats_v4 $B > /dev/null 2>&1
cat gpurun_out/probe.txt
ls -la gpurun_out
