#!/bin/bash
# A/B: bra pair bits in the sort key (0 / 2 / 3), task run length, c5 fourfold
python -m pytest tests/test_gpu_direct_twin.py -x -q -k c5 2>&1 | tail -40
for lib in libhxf_h0.so libhxf_h2.so; do
  for tb in 16 32; do
    echo "== $lib TASK_BLOCK=$tb"
    HXF_TASK_BLOCK=$tb HXF_LIB=$PWD/paper_1401_6961_b200/$lib python tools/step_breakdown.py c5 fourfold 2 2>&1 | tail -1
  done
done
