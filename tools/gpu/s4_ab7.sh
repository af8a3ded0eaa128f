#!/bin/bash
# leaf-screen grid (blocks per SM; 4 are resident) x task run length, c5 fourfold
run() { echo "== $*"; env "$@" python tools/step_breakdown.py c5 fourfold 2 2>&1 | tail -1; }
run HXF_SCREEN_BLOCKS=4 HXF_TASK_BLOCK=16
run HXF_SCREEN_BLOCKS=4 HXF_TASK_BLOCK=32
run HXF_SCREEN_BLOCKS=4 HXF_TASK_BLOCK=8
run HXF_SCREEN_BLOCKS=8 HXF_TASK_BLOCK=16
run HXF_SCREEN_BLOCKS=12 HXF_TASK_BLOCK=16
run HXF_SCREEN_BLOCKS=24 HXF_TASK_BLOCK=16
