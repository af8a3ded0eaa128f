set -x
mkdir -p gpurun_out
HXF_ERI_STATS=1 timeout 600 python tools/step_breakdown.py c5 fourfold 3 > gpurun_out/r2_step_v6.log 2>&1
tail -4 gpurun_out/r2_step_v6.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2_launches_v6.csv python tools/one_build.py c5 fourfold - 1 > gpurun_out/r2_ncu_v6.log 2>&1; echo ncu_rc=$?
timeout 900 python -m pytest tests/test_gpu_full_parity.py -x -q -k full_size > gpurun_out/r2_parity6.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_parity6.log
