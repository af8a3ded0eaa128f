#!/bin/bash
# screen / ERI overlap (HXF_PIPE=1: the screen of chunk i+1 beside the ERI stage of chunk i) with the screen
# grid cut to k blocks per SM so ERI blocks can be co-resident
run() { echo "== $*"; env "$@" python tools/step_breakdown.py c5 fourfold 2 2>&1 | tail -1; }
run HXF_PIPE=0
run HXF_PIPE=1
run HXF_PIPE=1 HXF_SCREEN_BLOCKS=2
run HXF_PIPE=1 HXF_SCREEN_BLOCKS=3
run HXF_PIPE=0 HXF_SCREEN_BLOCKS=2
run HXF_PIPE=0 HXF_SCREEN_BLOCKS=4
