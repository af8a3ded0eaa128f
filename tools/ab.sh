#!/bin/bash
# A/B of library variants on one GPU box: tools/ab.sh <config> <mode> <reps> lib1.so lib2.so ...
# (variants are built with make OUT=../libhxf_<tag>.so OBJDIR=../../build/obj_<tag> NVFLAGS="... -D...")
cfg=$1; mode=$2; reps=$3; shift 3
for lib in "$@"; do
  echo "== $lib"
  HXF_LIB=$PWD/paper_1401_6961_b200/$lib python tools/step_breakdown.py $cfg $mode $reps 2>&1 | tail -2
done
