#!/bin/bash
# Round evidence: headline bench (with CPU baseline), reference arm, every
# other config, the config-5 GIN batch sweep, products at batch 8000, and the
# launch list of the headline's profiled window.  Usage: tools/gpu_all.sh <tag>
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
nproc > $O/host.txt; free -g >> $O/host.txt
timeout 900 python bench.py > $O/bench_products.json 2> $O/bench_products.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
for c in reddit gin products_sage products_host; do
  timeout 900 python bench.py --config $c --steps 20 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --config products_host --cache-ratio 0.1 --steps 20 --no-cpu-baseline > $O/bench_products_host_c01.json 2> $O/bench_products_host_c01.err
for bs in 512 1024 2048 4096 8192; do
  timeout 600 python bench.py --config gin --bs $bs --steps 20 --no-cpu-baseline > $O/bench_gin_bs$bs.json 2> $O/bench_gin_bs$bs.err
done
timeout 600 python bench.py --bs 8000 --steps 20 --no-cpu-baseline > $O/bench_products_bs8000.json 2> $O/bench_products_bs8000.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches.csv python bench.py --profile --no-cpu-baseline > $O/prof.log 2>&1
timeout 1500 python bench.py --config papers --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_papers.json 2> $O/bench_papers.err
timeout 1500 python bench.py --config papers --cache-ratio 1.0 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_papers_c1.0.json 2> $O/bench_papers_c1.0.err
timeout 1500 python bench.py --config papers_hbm --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_papers_hbm.json 2> $O/bench_papers_hbm.err
for f in $O/bench_*.json; do python -c "
import json
d = json.loads(open('$f').read().strip().splitlines()[-1])
print('$f'.split('/')[-1], round(d['value'] / 1e9, 3), 'G', round(d.get('ms_per_step', 0), 3), 'ms', 'e2e', round(d.get('e2e', {}).get('value', 0) / 1e9, 3))
" 2>/dev/null || echo "$f failed"; done
