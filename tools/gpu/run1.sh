set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest1.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r2_pytest1.log
timeout 600 python tools/step_breakdown.py c5 fourfold 3 > gpurun_out/r2_step_base.log 2>&1
HXF_LIB=$PWD/var/libhxf_noatom.so timeout 600 python tools/step_breakdown.py c5 fourfold 3 > gpurun_out/r2_step_noatom.log 2>&1
cat gpurun_out/r2_step_base.log gpurun_out/r2_step_noatom.log
