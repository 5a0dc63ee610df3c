timeout 600 ncu --set full --import-source on --clock-control none -k regex:stats_strict -s 1 -c 1 -o gpurun_out/prof_sstats_$1 python bench.py --mode strict --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo > /dev/null 2>&1
ls gpurun_out | grep sstats
