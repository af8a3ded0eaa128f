#!/bin/bash
# round-2 session-4 measurement: bench lines, ncu launch list, DRAM pass, full captures (c5 fourfold)
tag=${1:-r02s4}
mkdir -p gpurun_out
python bench.py --impl reference > gpurun_out/${tag}_bench_c5_reference.json 2> gpurun_out/${tag}_bench_ref.err
python bench.py > gpurun_out/${tag}_bench_c5_fourfold.json 2> gpurun_out/${tag}_bench.err; echo bench_rc=$?
tail -c 600 gpurun_out/${tag}_bench_c5_fourfold.json
# launch list of one build (per-launch times are cold-cache and serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/${tag}_launches_c5.csv python tools/one_build.py c5 fourfold - 1 > gpurun_out/${tag}_ncu_launches.log 2>&1; echo launches_rc=$?
python tools/launch_stats.py gpurun_out/${tag}_launches_c5.csv 40 > gpurun_out/${tag}_launches_c5_summary.txt; head -12 gpurun_out/${tag}_launches_c5_summary.txt
# DRAM bytes per kernel family of one build
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_eri|k_screen2|k_expand|k_bin|DeviceRadixSort" --csv --log-file gpurun_out/${tag}_dram_launches_c5.csv python tools/one_build.py c5 fourfold - 1 > gpurun_out/${tag}_ncu_dram.log 2>&1; echo dram_rc=$?
python tools/ncu_dram.py gpurun_out/${tag}_dram_launches_c5.csv c5 fourfold 1 > gpurun_out/${tag}_ncu_c5_dram.json; head -c 1200 gpurun_out/${tag}_ncu_c5_dram.json
# full captures: leaf screen, (ss|ss) far and near
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_screen2" -s 8 -c 1 -o gpurun_out/${tag}_full_screen_c5 python tools/one_build.py c5 fourfold - 1 > gpurun_out/${tag}_full_screen.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_eri<.int.0, .int.0, .int.0, .int.0, .bool.1>" -s 8 -c 1 -o gpurun_out/${tag}_full_ssfar_c5 python tools/one_build.py c5 fourfold - 1 > gpurun_out/${tag}_full_ssfar.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_eri<.int.0, .int.0, .int.0, .int.0, .bool.0>" -s 8 -c 1 -o gpurun_out/${tag}_full_ssnear_c5 python tools/one_build.py c5 fourfold - 1 > gpurun_out/${tag}_full_ssnear.log 2>&1; echo rc=$?
gzip -f gpurun_out/${tag}_launches_c5.csv gpurun_out/${tag}_dram_launches_c5.csv
ls -la gpurun_out | tail -20
