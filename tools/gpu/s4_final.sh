#!/bin/bash
tag=${1:-r02s4e}
python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/${tag}_gputests.log; cat gpurun_out/${tag}_gputests.log
python __graft_entry__.py smoke 2>&1 | tail -1
python bench.py --impl reference > gpurun_out/${tag}_bench_c5_reference.json 2> gpurun_out/${tag}_bench_ref.err
python bench.py > gpurun_out/${tag}_bench_c5_fourfold.json 2> gpurun_out/${tag}_bench.err; echo bench_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/${tag}_launches_c5.csv python tools/one_build.py c5 fourfold - 1 > gpurun_out/${tag}_ncu_launches.log 2>&1; echo launches_rc=$?
python tools/launch_stats.py gpurun_out/${tag}_launches_c5.csv 40 > gpurun_out/${tag}_launches_c5_summary.txt; head -8 gpurun_out/${tag}_launches_c5_summary.txt
gzip -f gpurun_out/${tag}_launches_c5.csv
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_screen2" -s 8 -c 1 -o gpurun_out/${tag}_full_screen_c5 python tools/one_build.py c5 fourfold - 1 > gpurun_out/${tag}_full_screen.log 2>&1; echo rc=$?
