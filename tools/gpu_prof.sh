# usage: bash tools/gpu_prof.sh TAG  -> gpurun_out/prof_apply_TAG.ncu-rep
B="python bench.py --mode fast --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:apply_tc -s 3 -c 1 -o gpurun_out/prof_apply_$1 $B > /dev/null 2>&1
ls -la gpurun_out/prof_apply_$1.ncu-rep
