#!/bin/bash
# Interleaved A/B of bench.py: the working tree vs builds kept under
# _variants/<name>/ (bench.py + package with its .so).
# Usage: tools/ab_variants.sh rounds "bench args" name...
R=$1; shift; A=$1; shift
for i in $(seq $R); do
  for v in cur "$@"; do
    if [ "$v" = cur ]; then b=bench.py; else b=_variants/$v/bench.py; fi
    timeout 400 python $b $A --no-cpu-baseline > gpurun_out/abv.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/abv.json').read().strip().splitlines()[-1]); print('$v', '$A', round(d['value']/1e9,3), round(d['ms_per_step'],3), round(d['e2e']['value']/1e9,3))"
  done
done
