#!/bin/bash
# leaf-screen task runs handed out dynamically (HXF_SCREEN_DYN, default) against the static block-cyclic deal
run() { echo "== $*"; env "${@:3}" python tools/step_breakdown.py $1 $2 3 2>&1 | tail -1; }
run c5 fourfold HXF_SCREEN_DYN=1
run c5 fourfold HXF_SCREEN_DYN=0
run c5 fourfold HXF_SCREEN_DYN=1 HXF_TASK_BLOCK=32
run c5 fourfold HXF_SCREEN_DYN=1 HXF_TASK_BLOCK=64
run c4 fourfold HXF_SCREEN_DYN=1
run c4 naive HXF_SCREEN_DYN=1
python -m pytest tests/test_gpu_order_invariance.py tests/test_gpu_parity.py tests/test_gpu_ties.py -x -q 2>&1 | tail -3
