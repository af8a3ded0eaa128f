#!/bin/bash
# with dynamic runs: screen grid (blocks per SM; 4 resident)
run() { echo "== $*"; env "${@:3}" python tools/step_breakdown.py $1 $2 3 2>&1 | tail -1; }
run c5 fourfold HXF_SCREEN_BLOCKS=48
run c5 fourfold HXF_SCREEN_BLOCKS=4
run c5 fourfold HXF_SCREEN_BLOCKS=8
run c4 fourfold HXF_SCREEN_BLOCKS=48
run c4 fourfold HXF_SCREEN_BLOCKS=4
run c3 naive HXF_SCREEN_BLOCKS=32
run c3 naive HXF_SCREEN_BLOCKS=2
