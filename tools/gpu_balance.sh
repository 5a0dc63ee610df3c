# balanced pair ranges (prep, from measured CTA speeds) vs the even split
# (-DLOPT_EVEN_SPLIT), same box: apply time (ncu), per-CTA balance, step time
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout -s KILL 400 python -m pytest tests/test_gpu_fast.py tests/test_gpu_strict.py tests/test_gpu_graph.py -q -x 2>&1 | tail -2
bash tools/build_variant.sh /tmp/lopt_even.so -DLOPT_EVEN_SPLIT > /dev/null 2>&1
bash tools/build_variant.sh /tmp/lopt_cc.so -DLOPT_CTA_CLOCK > /dev/null 2>&1
bash tools/build_variant.sh /tmp/lopt_evencc.so -DLOPT_CTA_CLOCK -DLOPT_EVEN_SPLIT > /dev/null 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
for rep in 1 2; do
for v in even base; do
  so=/tmp/lopt_$v.so; [ $v = base ] && so=""
  LOPT_SO=$so timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"apply_pair" -s 3 -c 1 --csv $B 2>/dev/null | grep -E "apply_pair" | awk -F'","' -v n=$v '{print n, $5, $15}'
done
done
for v in evencc cc; do echo "== $v"; LOPT_SO=/tmp/lopt_$v.so timeout 200 python tools/cta_balance.py ${WL:-vit_b16} 2>&1 | head -8; done
for v in even base; do
  so=/tmp/lopt_$v.so; [ $v = base ] && so=""
  LOPT_SO=$so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-velo 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['roofline']['phase_ms'])"
done
