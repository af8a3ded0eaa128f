#!/bin/bash
# One line per BASELINE config and driver (run on the GPU box; output under gpurun_out/).
# usage: bash tools/bench_all.sh TAG
tag=${1:-all}
mkdir -p gpurun_out
for cfg in c1 c2 c3 c4; do
  for mode in naive fourfold; do
    timeout 900 python bench.py --config $cfg --mode $mode --steps 10 --warmup 3 \
      > gpurun_out/${tag}_bench_${cfg}_${mode}.json 2> gpurun_out/${tag}_bench_${cfg}_${mode}.err
    echo "$cfg $mode rc=$?" >> gpurun_out/${tag}_bench_all.rc
  done
done
