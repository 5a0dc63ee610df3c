B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_active.avg,gpc__cycles_elapsed.max --cache-control none --clock-control none -k regex:"apply_pair|prep_kernel|stats_fast|factor_part" -s 12 -c 8 $B 2>/dev/null | grep -E "apply_pair|prep_kernel|stats_fast|factor_part|duration|cycles"
bash tools/build_variant.sh /tmp/lopt_cc.so -DLOPT_CTA_CLOCK > /dev/null 2>&1
LOPT_SO=/tmp/lopt_cc.so timeout 200 python tools/cta_balance.py 2>&1 | head -1
