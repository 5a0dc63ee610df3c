# pair-kernel change check: fast parity (bounded), ncu of the apply kernel
timeout -s KILL 200 python -m pytest tests/test_gpu_fast.py tests/test_gpu_velo.py -x -q 2>&1 | tail -2 || exit 1
timeout -s KILL 300 bash tools/gpu_ncu_apply.sh 3 ${1:-r2_chk} | head -16
