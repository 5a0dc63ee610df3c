# factor partials kernel vs LOPT_FACTOR_TILE (same box), ViT-B/16 and GPT-2 medium
for wl in vit_b16 gpt2_medium; do
  for t in 65536 98304 114688 131072 163840 196608 262144; do
    LOPT_FACTOR_TILE=$t timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"factor_(partials|reduce)" -s 6 -c 2 --csv python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo 2>/dev/null | grep -E "factor_" | awk -F'","' -v w=$wl -v t=$t '{print w, t, $5, $15}'
  done
done
