set -x
mkdir -p gpurun_out
HXF_ERI_STATS=1 timeout 600 python tools/step_breakdown.py c5 fourfold 3 > gpurun_out/r2_step_far.log 2>&1
cat gpurun_out/r2_step_far.log
timeout 1800 python -m pytest tests/test_gpu_full_parity.py tests/test_gpu_parity.py -x -q -s > gpurun_out/r2_parity2.log 2>&1; echo rc=$?
tail -5 gpurun_out/r2_parity2.log
