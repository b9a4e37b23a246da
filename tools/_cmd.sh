timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python tools/time_kernels.py varlib/nat3.so varlib/ucon.so varlib/ucon_d20.so 2>&1
