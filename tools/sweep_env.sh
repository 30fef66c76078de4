#!/bin/bash
# A/B sweep of environment switches on the headline bench: one line per variant.
# Usage: tools/sweep_env.sh <tag> "VAR=a VAR2=b" "VAR=c" ...   ("" = defaults)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; shift; mkdir -p $O
i=0
for v in "$@"; do
  i=$((i+1))
  env $v timeout 600 python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > $O/v$i.json 2> $O/v$i.err
  python - "$v" $O/v$i.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"{sys.argv[1] or 'defaults':40s} {d['value']/1e9:.3f}G  {d['ms_per_step']:.3f} ms/win  e2e {d['e2e']['value']/1e9:.3f}G", flush=True)
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
