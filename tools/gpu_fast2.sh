set -x
timeout 600 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_fast.py -x -q -s 2>&1 | grep -E "relL2|elementwise|passed|failed|Error|assert" | head -40
LOPT_BENCH_MODE=fast timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -2
LOPT_BENCH_MODE=fast timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lopt -c 40 --csv --log-file gpurun_out/launches_fast.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/launches_fast.csv")))
hdr = [r for r in rows if r and r[0] == "ID"]
for r in rows:
    if r and r[0].isdigit():
        print(r[4][:60], r[7], r[8], r[-1])
PY
