# factor partials A/B: the committed source vs a variant build ($VARIANTS as in
# tools/gpu_ncu_variants.sh), same box, ViT-B/16 and GPT-2 medium
timeout -s KILL 300 python -m pytest tests/test_gpu_fast.py tests/test_gpu_strict.py -q -x 2>&1 | tail -1
for v in $VARIANTS; do
  name=${v%%:*}; flags=${v#*:}
  bash tools/build_variant.sh /tmp/lopt_$name.so lopt_factors.cu $(echo $flags | tr ',' ' ') > /dev/null 2>&1 || echo "$name build failed"
done
for rep in 1 2; do for v in base $VARIANTS; do name=${v%%:*}; so=/tmp/lopt_$name.so; [ $name = base ] && so=""
for wl in vit_b16 gpt2_medium; do
LOPT_SO=$so timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"factor_partials" -s 3 -c 1 --csv python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo 2>/dev/null | grep factor_partials | awk -F'","' -v n=$name -v w=$wl '{print n, w, $15}'
done; done; done
