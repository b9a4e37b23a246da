timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python tools/time_kernels.py varlib/s36d24.so varlib/d24e16.so 2>&1
python bench.py --no-e2e --no-cpu > gpurun_out/b.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print(d['value'], r['compress_gbs'], r['decompress_gbs'], r['step_frac'], d['async_insitu']['slowdown'])"
