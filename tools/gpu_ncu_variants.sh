# same-box ncu A/B of kernel builds: base + variants given as "name:-DFLAGS" ($VARIANTS);
# $KERNEL (regex, default apply_pair) and $SRC (the recompiled source) select the kernel
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
run() {
  for rep in 1 2; do
    LOPT_SO=$2 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"${KERNEL:-apply_pair}" -s 3 -c 1 --csv $B 2>/dev/null | grep -E "${KERNEL:-apply_pair}" | awk -F'","' -v n=$1 '{printf "%s %s %s\n", n, $13, $15}'
  done
}
run base ""
for v in $VARIANTS; do
  name=${v%%:*}; flags=${v#*:}
  bash tools/build_variant.sh /tmp/lopt_$name.so ${SRC:-lopt_apply_tc.cu} $(echo $flags | tr ',' ' ') || { echo "$name build failed"; continue; }
  LOPT_SO=/tmp/lopt_$name.so timeout -s KILL 200 python -m pytest tests/test_gpu_fast.py -q -x 2>&1 | tail -1
  run $name /tmp/lopt_$name.so
done
run base_again ""
