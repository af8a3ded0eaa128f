set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s2b_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/s2b_pytest.log
HXF_ERI_STATS=1 ONE_BUILD_CLASSES=1 timeout 600 python tools/step_breakdown.py c5 fourfold 3 > gpurun_out/s2b_step.log 2>&1
cat gpurun_out/s2b_step.log
for k in "0, .int.0, .int.0, .int.0, .bool.1" "0, .int.0, .int.0, .int.0, .bool.0" "0, .int.1, .int.0, .int.0, .bool.1"; do
  tag=$(echo "$k" | tr -cd '01')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_eri<.int.$k>" -s 8 -c 1 -o gpurun_out/s2b_eri_$tag python tools/one_build.py c5 fourfold - 1 > gpurun_out/s2b_eri_$tag.log 2>&1; echo ncu_rc=$?
done
