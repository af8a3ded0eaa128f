set -x
mkdir -p gpurun_out
K='regex:k_screen2'
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K" -s 8 -c 1 -o gpurun_out/r2_full_screen_c5 python tools/one_build.py c5 fourfold - 1 > gpurun_out/r2_full_screen.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_eri<.int.0, .int.0, .int.0, .int.0, .bool.1>" -s 8 -c 1 -o gpurun_out/r2_full_ssfar_c5 python tools/one_build.py c5 fourfold - 1 > gpurun_out/r2_full_ssfar.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_eri<.int.0, .int.0, .int.0, .int.0, .bool.0>" -s 8 -c 1 -o gpurun_out/r2_full_ssnear_c5 python tools/one_build.py c5 fourfold - 1 > gpurun_out/r2_full_ssnear.log 2>&1; echo rc=$?
ls -la gpurun_out
