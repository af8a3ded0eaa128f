#!/bin/bash
# ERI class kernels dealt over 1 / 2 / 4 streams, c5 and c4 fourfold
run() { echo "== $*"; env "${@:3}" python tools/step_breakdown.py $1 $2 3 2>&1 | tail -1; }
run c5 fourfold HXF_ERI_STREAMS=1
run c5 fourfold HXF_ERI_STREAMS=2
run c5 fourfold HXF_ERI_STREAMS=4
run c4 fourfold HXF_ERI_STREAMS=1
run c4 fourfold HXF_ERI_STREAMS=4
run c3 naive HXF_ERI_STREAMS=1
run c3 naive HXF_ERI_STREAMS=4
python -m pytest tests/test_gpu_order_invariance.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
