timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python tools/time_kernels.py varlib/tthr.so varlib/pdl.so 2>&1
python bench.py --no-e2e --no-cpu --no-async > gpurun_out/b_pdl.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/b_pdl.json')); r=d['roofline']; print(d['value'], r['compress_gbs'], r['decompress_gbs'], r['step_frac'])"
