# A/B products bench: env settings given as args ("-" = default)
for e in "$@"; do
  if [ "$e" = "-" ]; then env_s=""; else env_s="$e"; fi
  env $env_s timeout 400 python bench.py --steps 40 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$e', round(d['value']/1e9,3), round(d['ms_per_step'],3), round(d['e2e']['value']/1e9,3))"
done
