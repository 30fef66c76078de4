#!/bin/bash
# all bench configs once (1 GPU); papers last (largest, host features)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
free -g > $O/mem.txt 2>&1; nproc >> $O/mem.txt
for c in reddit gin products_sage products_host; do
  timeout 900 python bench.py --config $c --steps 10 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  echo "$c rc=$?"
done
timeout 900 python bench.py --config products_host --cache-ratio 0.1 --steps 10 --no-cpu-baseline > $O/bench_products_host_c01.json 2> $O/bench_products_host_c01.err; echo "cache rc=$?"
timeout 1500 python bench.py --config papers --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_papers.json 2> $O/bench_papers.err; echo "papers rc=$?"
for f in $O/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,1), 'M edges/s', round(d['ms_per_step'],3), 'ms', d.get('stages_ms_per_step'))" 2>/dev/null || echo "$f failed"; done
tail -3 $O/bench_papers.err
