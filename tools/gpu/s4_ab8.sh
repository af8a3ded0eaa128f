#!/bin/bash
run() { echo "== $*"; env "${@:3}" python tools/step_breakdown.py $1 $2 3 2>&1 | tail -1; }
run c4 naive HXF_SCREEN_BLOCKS=8
run c4 naive HXF_SCREEN_BLOCKS=32
run c4 naive HXF_SCREEN_BLOCKS=64
run c4 fourfold HXF_SCREEN_BLOCKS=12
run c4 fourfold HXF_SCREEN_BLOCKS=48
run c3 fourfold HXF_SCREEN_BLOCKS=12
run c3 fourfold HXF_SCREEN_BLOCKS=48
run c5 fourfold HXF_SCREEN_BLOCKS=48
run c5 fourfold HXF_SCREEN_BLOCKS=44
run c5 fourfold HXF_SCREEN_BLOCKS=52
run c5 fourfold HXF_SCREEN_BLOCKS=60
