timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python tools/time_kernels.py varlib/bk.so 2>&1
ISF_LOSSY_LIB=varlib/bk.so timeout 300 python tools/lx_sweep.py 2>&1 | python -c "
import json,sys; d=json.load(sys.stdin); [print(k, round(v['compress_gbs']), round(v['decompress_gbs'])) for k,v in d.items() if 'lx8' in k]"
ISF_LOSSY_LIB=varlib/pst.so true
