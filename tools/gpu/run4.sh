set -x
mkdir -p gpurun_out
for v in default farb2 nofar; do
  if [ $v = default ]; then L=""; else L=$PWD/var/libhxf_$v.so; fi
  HXF_LIB=$L HXF_ERI_STATS=1 timeout 600 python tools/step_breakdown.py c5 fourfold 3 > gpurun_out/r2_step_$v.log 2>&1
  tail -3 gpurun_out/r2_step_$v.log
done
HXF_LIB=$PWD/var/libhxf_profscreen.so timeout 600 python tools/step_breakdown.py c5 fourfold 2 > gpurun_out/r2_step_profscreen.log 2>&1
tail -6 gpurun_out/r2_step_profscreen.log
timeout 900 python -m pytest tests/test_gpu_full_parity.py -x -q -s -k "full_size" > gpurun_out/r2_parity3.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2_parity3.log
