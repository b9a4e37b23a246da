python tools/time_kernels.py varlib/cur.so varlib/d20.so varlib/d24.so varlib/d12.so 2>&1
