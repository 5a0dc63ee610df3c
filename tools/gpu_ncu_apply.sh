# ncu --set full of one apply launch (variant $1, tag $2) + the opcode summary
V=${1:-2}; TAG=${2:-v}
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-velo"
LOPT_APPLY_VARIANT=$V timeout 900 ncu --set full --import-source on --clock-control none -k regex:"apply_[a-z]+_kernel" -s 3 -c 1 -o gpurun_out/prof_apply_$TAG $B > gpurun_out/ncu_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_apply_$TAG.ncu-rep > gpurun_out/prof_apply_${TAG}_summary.txt 2>&1
head -60 gpurun_out/prof_apply_${TAG}_summary.txt
