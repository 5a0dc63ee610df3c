# layer-3 weights from the launch parameter (uniform registers) vs the operand image (LOPT_NO_W3C=1)
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout -s KILL 600 python -m pytest tests/test_gpu_fast.py tests/test_gpu_strict.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
for rep in 1 2; do for v in 0 1; do
  E=""; [ $v = 1 ] && E="LOPT_NO_W3C=1"
  env $E timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:apply_pair -s 3 -c 1 --csv $B 2>/dev/null | grep apply_pair | awk -F'","' -v n=no_w3c=$v '{print n, $13, $15}'
done; done
for v in 0 1; do E=""; [ $v = 1 ] && E="LOPT_NO_W3C=1"
  env $E timeout 300 python bench.py --steps 30 --warmup 10 --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no_w3c=$v', round(d['ms_per_step'],4), d['step_ms_p10_p50_p90'], {k: round(x,4) for k,x in d['roofline']['phase_ms'].items()})"
done
