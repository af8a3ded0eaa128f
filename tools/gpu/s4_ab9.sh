#!/bin/bash
run() { echo "== $*"; env "$@" python tools/step_breakdown.py c5 fourfold 2 2>&1 | tail -1; }
L=$PWD/paper_1401_6961_b200
run HXF_LIB=$L/libhxf_b4.so HXF_BIN_BLOCKS=48
run HXF_LIB=$L/libhxf_b48.so HXF_BIN_BLOCKS=24
run HXF_LIB=$L/libhxf_b48.so HXF_BIN_BLOCKS=48
run HXF_LIB=$L/libhxf_b28.so HXF_BIN_BLOCKS=24
run HXF_LIB=$L/libhxf_b28.so HXF_BIN_BLOCKS=48
