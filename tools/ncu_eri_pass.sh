#!/bin/bash
# ncu evidence for the ERI stage (run on the GPU box; outputs under gpurun_out/):
#  1. FP64 instruction counts of every k_eri launch of one c4 fourfold build
#     (-> tools/fp64_rate.py -> executed flops per primitive quartet per class)
#  2. one --set full capture of the (ss|ss) kernel (the top kernel)
tag=${1:-eri}
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum
ONE_BUILD_CLASSES=1 timeout 900 ncu --metrics $M --clock-control none -k regex:"k_eri" --csv \
  --log-file gpurun_out/${tag}_fp64_c4.csv python tools/one_build.py c4 fourfold - 1 \
  > gpurun_out/${tag}_fp64_c4.log 2>&1
echo "fp64 rc=$?" >> gpurun_out/${tag}_ncu.rc
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_eri<.int.0, .int.0, .int.0, .int.0>" -s 2 -c 1 \
  -o gpurun_out/${tag}_full_ssss_c4 python tools/one_build.py c4 fourfold - 1 > gpurun_out/${tag}_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${tag}_ncu.rc
