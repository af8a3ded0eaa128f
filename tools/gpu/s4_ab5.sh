#!/bin/bash
# ERI occupancy re-tune after the locality changes (min blocks per SM: far (ss|ss) / far p classes / near (ss|ss))
for lib in libhxf_f6.so libhxf_f8.so libhxf_f6p4.so libhxf_f6n2.so; do
  echo "== $lib"
  HXF_LIB=$PWD/paper_1401_6961_b200/$lib python tools/step_breakdown.py c5 fourfold 2 2>&1 | tail -1
done
