timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python tools/time_kernels.py varlib/cur.so varlib/exs.so 2>&1
ncu --set full --import-source on --clock-control none -k regex:decompress8 -s 1 -c 1 -o gpurun_out/d8x python tools/time_kernels.py varlib/exs.so > /dev/null 2>&1
