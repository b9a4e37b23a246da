timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 100 python tools/time_kernels.py paper_2407_20731_b200/libisf_lossy.so 2>&1
