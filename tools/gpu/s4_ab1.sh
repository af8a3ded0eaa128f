#!/bin/bash
# A/B: leaf-task order (HXF_LEAF_SORT) x block-cyclic screen runs (HXF_TASK_BLOCK), c5 fourfold
for v in "1 32" "0 32" "1 1" "0 1" "1 8" "1 128" "1 512"; do
  set -- $v
  echo "== LEAF_SORT=$1 TASK_BLOCK=$2"
  HXF_LEAF_SORT=$1 HXF_TASK_BLOCK=$2 python tools/step_breakdown.py c5 fourfold 2 2>&1 | tail -1
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_digest.py -x -q 2>&1 | tail -3
