#!/bin/bash
# select A/B: sampler parity tests, standalone sampler window time and the
# headline bench per variant.  Usage: tools/gpu_sel.sh <tag> "ENV=a" "ENV=b" ...
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; shift; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_scale.py tests/test_gpu_configs.py -q -x -k "sampl or window or scale or khop or hub or frontier" > $O/test.log 2>&1; tail -2 $O/test.log
for v in "$@"; do
  env $v timeout 300 python tools/bench_stages.py --windows 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', 'sampler ms/window', round(d['sampler_ms_per_window'],3), 'draws', d['draws_per_window'])"
done
STEPS=60 bash tools/sweep_env.sh $(basename $O)-bench "$@"
