#!/bin/bash
# bench + launch list of the timed steps (one GPU)
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 600 python bench.py --no-cpu-baseline ${2:-} > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches.csv python bench.py --profile --no-cpu-baseline ${2:-} > $O/prof.log 2>&1
python profiles/summarize_launches.py $O/launches.csv 0 45 > $O/launches_summary.txt
cat $O/bench.json; cat $O/launches_summary.txt
