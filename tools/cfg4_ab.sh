# cfg4 sweep of alternative builds on the same box (dev tool): tools/cfg4_ab.sh "label|ENV=val" ...
for spec in "$@"; do
  lab=${spec%%|*}; envs=${spec#*|}
  env $envs python bench.py --no-e2e --no-cpu --no-async --no-parity --steps 5 > gpurun_out/var4.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/var4.json'))
print('$lab', ' '.join(f\"lx{c['lx']}/{c['eps']:.0e}:{round(c['compress_gbs'])}/{round(c['decompress_gbs'])}\" for c in d['cfg4']))"
done
