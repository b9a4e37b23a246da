timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
python tools/time_kernels.py varlib/early.so 2>&1
ISF_LOSSY_LIB=varlib/early.so timeout 600 python tools/lx_sweep.py 2>&1 | python -c "
import json,sys; d=json.load(sys.stdin); [print(k, round(v['compress_gbs']), round(v['decompress_gbs'])) for k,v in d.items() if 'lx8' in k]"
