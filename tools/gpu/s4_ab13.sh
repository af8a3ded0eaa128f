#!/bin/bash
run() { echo "== $*"; env "${@:3}" python tools/step_breakdown.py $1 $2 3 2>&1 | tail -1; }
L=$PWD/paper_1401_6961_b200
run c5 fourfold HXF_LIB=$L/libhxf.so
run c5 fourfold HXF_LIB=$L/libhxf_f7.so
run c5 fourfold HXF_LIB=$L/libhxf_f5p3.so
run c5 fourfold HXF_LIB=$L/libhxf.so HXF_TASK_BLOCK=48
