timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
ISF_LOSSY_LIB=varlib/gc2.so timeout 300 python tools/lx_sweep.py 2>&1 | python -c "
import json,sys; d=json.load(sys.stdin); [print(k, round(v['compress_gbs']), round(v['decompress_gbs'])) for k,v in d.items()]"
