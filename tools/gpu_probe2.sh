python tools/probe_umma.py
timeout 600 python -m pytest tests/test_gpu_velo.py tests/test_gpu_fast.py tests/test_gpu_strict.py -x -q 2>&1 | tail -15
