#!/bin/bash
for bb in 5 3 2; do echo "== BIN_BLOCKS=$bb"; HXF_BIN_BLOCKS=$bb python tools/step_breakdown.py c5 fourfold 2 2>&1 | tail -1; done
