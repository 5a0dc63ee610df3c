# build_variant.sh OUT.so [SRC.cu[,SRC2.cu...]] "-DFLAG=..." -- the library with
# the given sources (default lopt_apply_tc.cu) recompiled under extra defines
# (tuning experiments; load with LOPT_SO=OUT.so)
set -e
OUT=$1; shift
SRCS=lopt_apply_tc.cu
case "$1" in *.cu) SRCS=$1; shift;; esac
D=$(dirname "$0")/../paper_2506_10315_b200
OBJ=$(mktemp -d)
OTHERS=$(ls $D/_lib/obj/*.o)
for SRC in $(echo $SRCS | tr ',' ' '); do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC -I $D/../include "$@" -c $D/csrc/$SRC -o $OBJ/${SRC%.cu}.o
  OTHERS=$(echo "$OTHERS" | tr ' ' '\n' | grep -v "/${SRC%.cu}.o$")
done
nvcc -shared -o $OUT $OBJ/*.o $OTHERS -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -lcudart_static
