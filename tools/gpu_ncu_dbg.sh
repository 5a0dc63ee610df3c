# same-box ncu A/B of the apply kernel over LOPT_APPLY_DEBUG values ($DBGS): duration, IPC, instructions/element
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
for d in ${DBGS:-0 1 2 3}; do
  for rep in 1 2; do
    LOPT_APPLY_DEBUG=$d timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed.avg.per_cycle_active --clock-control none -k regex:"apply_pair" -s 3 -c 1 --csv $B 2>/dev/null | grep apply_pair | awk -F'","' -v d=$d '{printf "dbg %s %s %s\n", d, $13, $15}'
  done
done
