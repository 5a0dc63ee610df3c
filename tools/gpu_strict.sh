# Strict (bitwise) path: parity suites + strict bench line (+ optional ncu of strict apply/stats)
timeout 900 python -m pytest tests/test_gpu_strict.py tests/test_gpu_checkpoint.py tests/test_gpu_fullsize.py tests/test_gpu_velo.py -x -q 2>&1 | tail -3
timeout 300 python bench.py --mode strict --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'].get('phase_ms'))"
if [ -n "$1" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:strict_kernel -s 2 -c 2 -o gpurun_out/prof_strict_$1 python bench.py --mode strict --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo > /dev/null 2>&1
fi
