#!/bin/bash
# Build a variant of libemfgpu.so with extra nvcc defines (launch-bound /
# layout experiments): tools/build_variant.sh NAME -DFOO=1 ...
# Output: paper_2408_12479_b200/lib/var_NAME.so (git-ignored; travels with gpurun)
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2408_12479_b200/csrc
OUT=/tmp/var_$NAME; mkdir -p $OUT
make -s -C $SRC -j16 >/dev/null 2>&1
for f in $SRC/inst_*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" -c $f -o $OUT/$b.o 2>/dev/null &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/paper_2408_12479_b200/lib/var_$NAME.so \
  $(ls $ROOT/paper_2408_12479_b200/build/*.o | grep -v /inst_) $OUT/*.o
echo built var_$NAME.so
