# round 2: compute-sanitizer over the pair kernel paths (incl. peer staging), then a soak
timeout -s KILL 800 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 python -m pytest tests/test_gpu_fast.py -x -q -k "steps_vs_oracle and mlp and small_fc" 2>&1 | tail -3
timeout -s KILL 800 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 10 python -m pytest tests/test_gpu_fast.py -x -q -k "peer_bulk and 1" 2>&1 | tail -3
timeout -s KILL 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_fast.py tests/test_gpu_baselines.py -x -q -k "steps_vs_oracle or peer or adam or adafactor" 2>&1 | tail -3
timeout -s KILL 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_strict.py tests/test_gpu_velo.py -x -q 2>&1 | tail -3
timeout -s KILL 900 python tools/soak.py 1000 2>&1 | tail -5
