# build_variant.sh OUT.so "-DFLAG=..." -- the library with lopt_apply_tc.cu
# recompiled under extra defines (tuning experiments; load with LOPT_SO=OUT.so)
set -e
OUT=$1; shift
D=$(dirname "$0")/../paper_2506_10315_b200
OBJ=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -I $D/../include "$@" -c $D/csrc/lopt_apply_tc.cu -o $OBJ/apply.o
OTHERS=$(ls $D/_lib/obj/*.o | grep -v lopt_apply_tc.o)
nvcc -shared -o $OUT $OBJ/apply.o $OTHERS -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -lcudart_static
