#!/bin/bash
# On the GPU box: time each gpurun_ab/* variant with tools/tc_perf.py (args passed through),
# restoring the product library afterwards.  tools/ab_run.sh ROUNDS N ITERS MATH
ROOT=$(cd "$(dirname "$0")/.." && pwd)
LIB=$ROOT/paper_2511_23227_b200/libnpcg.so
cp $LIB /tmp/libnpcg.product.so
for r in $(seq 1 ${1:-1}); do
  for d in $ROOT/gpurun_ab/*/; do
    cp $d/libnpcg.so $LIB
    echo "== $(basename $d) round $r"
    timeout 300 python $ROOT/tools/tc_perf.py ${2:-1000000} ${3:-5} ${4:-bf16} 2>&1 | grep "step\|conv_"
  done
done
cp /tmp/libnpcg.product.so $LIB
