B="python bench.py --mode strict --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
timeout 300 python bench.py --mode strict --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('phase_ms'))"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:apply_strict -s 1 -c 1 -o gpurun_out/prof_strict_$1 $B > /dev/null 2>&1
ls gpurun_out | tail -3
