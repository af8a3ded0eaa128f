set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 2400 python -m pytest tests/test_gpu_full_parity.py tests/test_gpu_parity.py -k "full_size or tau_sweep or prim_neglect or unreached" -x -q -s > gpurun_out/r2_parity1.log 2>&1; echo rc=$?
tail -30 gpurun_out/r2_parity1.log
