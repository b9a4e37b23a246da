timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python tools/time_kernels.py varlib/nat3.so varlib/nat4.so 2>&1
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -k regex:"compact8" -c 4 python tools/time_kernels.py varlib/nat4.so 2>&1 | grep -E "duration"
