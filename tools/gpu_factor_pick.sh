# factor partials: per-plan tile pick + largest-first items vs the fixed 128 K tile
timeout -s KILL 300 python -m pytest tests/test_gpu_fast.py tests/test_gpu_strict.py -q -x 2>&1 | tail -1
for wl in vit_b16 gpt2_medium; do
for t in pick 131072; do
  E=""; [ $t != pick ] && E="LOPT_FACTOR_TILE=$t"
  env $E timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"factor_partials" -s 3 -c 2 python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo 2>/dev/null | grep -E "factor_partials|duration" | paste - - | awk -v w=$wl -v t=$t '{print w, t, $2, $(NF)}'
done
done
