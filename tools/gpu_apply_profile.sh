timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_velo.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py tests/test_gpu_strict.py -x -q 2>&1 | tail -4
for k in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('phase_ms'))"; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:apply_tc -s 3 -c 1 -o gpurun_out/prof_apply_$1 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo > /dev/null 2>&1
ls gpurun_out | grep $1
