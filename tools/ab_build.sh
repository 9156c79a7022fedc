#!/bin/bash
# A/B variants of libnpcg.so: tools/ab_build.sh NAME "-DFOO=1 -DBAR=2"
# builds gpurun_ab/NAME/libnpcg.so (the other objects from the normal build).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; DEFS=$2
OUT=$ROOT/gpurun_ab/$NAME; mkdir -p $OUT
python -m paper_2511_23227_b200.build >/dev/null
OBJS=$(ls $ROOT/paper_2511_23227_b200/_build/*.o | grep -v conv_tc.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O2 \
  -I$ROOT/include -I$ROOT/paper_2511_23227_b200/csrc $DEFS -c $ROOT/paper_2511_23227_b200/csrc/conv_tc.cu -o $OUT/conv_tc.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libnpcg.so $OBJS $OUT/conv_tc.o -lcuda
echo built $OUT/libnpcg.so
