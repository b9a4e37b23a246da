ncu --set full --import-source on --clock-control none -k regex:decompress8 -s 1 -c 1 -o gpurun_out/d8y python tools/time_kernels.py varlib/pdl.so > /dev/null 2>&1
