#!/bin/bash
# stable counting sort by ERI bin (replaces the CUB radix sort)
python tools/step_breakdown.py c5 fourfold 2 2>&1 | tail -1
python tools/step_breakdown.py c4 fourfold 3 2>&1 | tail -1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_digest.py tests/test_gpu_direct_twin.py -x -q 2>&1 | tail -15
