# build_variant.sh OUT.so [SRC.cu] "-DFLAG=..." -- the library with one source
# (default lopt_apply_tc.cu) recompiled under extra defines (tuning
# experiments; load with LOPT_SO=OUT.so)
set -e
OUT=$1; shift
SRC=lopt_apply_tc.cu
case "$1" in *.cu) SRC=$1; shift;; esac
D=$(dirname "$0")/../paper_2506_10315_b200
OBJ=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -I $D/../include "$@" -c $D/csrc/$SRC -o $OBJ/variant.o
OTHERS=$(ls $D/_lib/obj/*.o | grep -v "/${SRC%.cu}.o")
nvcc -shared -o $OUT $OBJ/variant.o $OTHERS -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -lcudart_static
