# time alternative in-tree builds of the library on the same box (dev tool)
for v in "$@"; do
  ISF_LOSSY_LIB=$v python bench.py --no-e2e --no-cpu --no-async --steps 20 > gpurun_out/var.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/var.json')); r=d['roofline']; print('$v', round(d['value']), round(r['compress_gbs']), round(r['decompress_gbs']))"
done
