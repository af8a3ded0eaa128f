#!/bin/bash
# leaf-screen grid (blocks per SM; 4 are resident) x task run length, c5 fourfold
run() { echo "== $*"; env "$@" python tools/step_breakdown.py c5 fourfold 2 2>&1 | tail -1; }
run HXF_SCREEN_BLOCKS=48 HXF_TASK_BLOCK=16
run HXF_SCREEN_BLOCKS=96 HXF_TASK_BLOCK=16
run HXF_SCREEN_BLOCKS=192 HXF_TASK_BLOCK=16
run HXF_SCREEN_BLOCKS=96 HXF_TASK_BLOCK=32
run HXF_SCREEN_BLOCKS=36 HXF_TASK_BLOCK=16
