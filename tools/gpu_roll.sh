# rolling apply kernel: parity (bounded), phase A/B vs the pair kernel, ncu
LOPT_APPLY_VARIANT=4 timeout -s KILL 150 python -m pytest tests/test_gpu_fast.py -x -q 2>&1 | tail -2 || exit 1
LOPT_APPLY_VARIANT=4 timeout -s KILL 240 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_velo.py -x -q 2>&1 | tail -2
timeout -s KILL 200 python tools/apply_ab.py LOPT_APPLY_VARIANT=4 LOPT_APPLY_VARIANT=3 2>&1 | tail -2
timeout -s KILL 200 bash tools/gpu_ncu_apply.sh 4 r2_roll1 | head -16
