set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s2a_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/s2a_pytest.log
timeout 1200 python bench.py > gpurun_out/s2a_bench.json 2> gpurun_out/s2a_bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/s2a_bench.json
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_screen2" -s 8 -c 1 -o gpurun_out/s2a_full_screen_c5 python tools/one_build.py c5 fourfold - 1 > gpurun_out/s2a_full_screen.log 2>&1; echo rc=$?
