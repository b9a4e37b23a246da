for v in "" build/var/lib_c12.so build/var/lib_c8.so build/var/lib_c20.so; do
  ISF_LOSSY_LIB=$v python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/var.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/var.json')); r=d['roofline']; print('$v', round(d['value']), round(r['compress_gbs']), round(r['decompress_gbs']))"
done
