# A/B timing of environment switches: bash tools/cmp_env.sh "ENV=1" "ENV=2" ...
i=0
for e in "$@"; do
  env $e timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b$i.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/b$i.log').read().strip().splitlines()[-1]);print('$e', round(d['ms_per_step'],4), ' '.join(k+'='+str(round(v['ms_per_launch']*v['launches_per_step'],4)) for k,v in d['kernels'].items()))"
  i=$((i+1))
done
