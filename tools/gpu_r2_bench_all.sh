# Round-2 bench lines: default, strict, GPT-2 medium VeLO (config 5), reference arm
set -x
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r2c.json
timeout 300 python bench.py --mode strict --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/bench_r2_strict.json
timeout 600 python bench.py --workload gpt2_medium --feature-set velo --no-cpu --no-e2e --no-velo --steps 10 2>&1 | tail -1 > gpurun_out/bench_r2_gpt2_velo.json
timeout 600 python bench.py --impl reference 2>&1 | tail -1 > gpurun_out/bench_r2_reference.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2c.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo > /dev/null 2>&1
LOPT_PEER_SCALAR=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"apply_pair" -s 3 -c 1 -o gpurun_out/prof_peers7_scalar python tools/peer_probe.py 7 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_peers7_scalar.ncu-rep > gpurun_out/prof_peers7_scalar_summary.txt 2>&1
cut -c1-400 gpurun_out/bench_r2*.json
grep "warp instructions" gpurun_out/prof_peers7_scalar_summary.txt
