# stats pass with the picked chunk vs the fixed 8 K chunk, ViT-B/16 and GPT-2 medium (same box)
for wl in vit_b16 gpt2_medium; do
  for fx in "" 1; do
    for rep in 1 2; do
      LOPT_STAT_CHUNK_FIXED=$fx timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:stats_fast -s 3 -c 1 --csv python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo 2>/dev/null | grep stats_fast | awk -F'","' -v w=$wl -v f="fixed=$fx" '{print w, f, $15}'
    done
  done
done
