# compute-sanitizer passes over the device paths (small cases)
timeout 800 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 python -m pytest tests/test_gpu_fast.py -x -q -k "steps_vs_oracle and mlp and small_fc" 2>&1 | tail -2
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_strict.py tests/test_gpu_velo.py -x -q 2>&1 | tail -2
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_fast.py -x -q -k "steps_vs_oracle and mlp and small_fc" 2>&1 | tail -2
