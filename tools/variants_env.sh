# time alternative builds / env settings on the same box (dev tool):
#   tools/variants_env.sh "label|ENV=val ENV2=val" ...   (ISF_LOSSY_LIB selects a build)
for spec in "$@"; do
  lab=${spec%%|*}; envs=${spec#*|}
  env $envs python bench.py --no-e2e --no-cpu --no-async --no-cfg4 --no-parity --steps 20 > gpurun_out/var.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/var.json')); r=d['roofline']; print('$lab', round(d['value']), round(r['compress_gbs']), round(r['decompress_gbs']), round(r['step_frac'],4), round(r['decompress_ms_per_field']*1000,1))"
done
