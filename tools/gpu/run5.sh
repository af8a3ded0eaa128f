set -x
mkdir -p gpurun_out
HXF_ERI_STATS=1 timeout 600 python tools/step_breakdown.py c5 fourfold 3 > gpurun_out/r2_step_v5.log 2>&1
tail -4 gpurun_out/r2_step_v5.log
timeout 1500 python -m pytest tests/test_gpu_full_parity.py tests/test_gpu_parity.py tests/test_gpu_reference_suite.py -x -q > gpurun_out/r2_parity5.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_parity5.log
