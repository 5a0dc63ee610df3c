# co-residency probe (tools/overlap_probe.py) for the base library and builds
# whose apply kernel leaves registers for a co-resident stats CTA
python tools/overlap_probe.py 2>&1 | tail -1 | sed 's/^/base /'
for v in "r112s128:-DLOPT_APPLY_MAXNREG=112,-DLOPT_STAT_THREADS=128,-DLOPT_STAT_MINB=8" \
         "r104s128:-DLOPT_APPLY_MAXNREG=104,-DLOPT_STAT_THREADS=128,-DLOPT_STAT_MINB=8"; do
  name=${v%%:*}; flags=${v#*:}
  bash tools/build_variant.sh /tmp/lopt_$name.so lopt_apply_tc.cu,lopt_fast.cu $(echo $flags | tr ',' ' ') > /dev/null 2>&1 || { echo "$name build failed"; continue; }
  LOPT_SO=/tmp/lopt_$name.so timeout -s KILL 200 python -m pytest tests/test_gpu_fast.py -q -x 2>&1 | tail -1
  LOPT_SO=/tmp/lopt_$name.so timeout -s KILL 200 python tools/overlap_probe.py 2>&1 | tail -1 | sed "s/^/$name /"
done
