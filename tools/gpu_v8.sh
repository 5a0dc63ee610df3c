# apply v8: parity, bench, launch list, full ncu capture of the apply kernel
set -x
B="python bench.py --mode fast --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_velo.py tests/test_gpu_dist.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --mode fast --steps 20 --warmup 5 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_v8.json
cut -c1-1200 gpurun_out/bench_v8.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v8.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:apply_tc -s 3 -c 1 -o gpurun_out/prof_apply_v8 $B > /dev/null 2>&1
ls gpurun_out
