#!/bin/bash
# One GPU session: build check, gpu tests, bench, launch list of the timed steps.
set -x
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches.csv python bench.py --profile --no-cpu-baseline > $O/prof.log 2>&1
tail -3 $O/pytest_gpu.log; cat $O/bench.json
