#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_scale.py tests/test_gpu_train.py -x -q > $O/test.log 2>&1; echo "rc=$?" >> $O/test.log
tail -3 $O/test.log
timeout 300 python tools/bench_stages.py --windows 10 > $O/stages.json 2>&1; cat $O/stages.json | tail -1
FGL_SELECT=tau timeout 300 python tools/bench_stages.py --windows 10 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select -c 6 python tools/bench_stages.py --windows 2 2>&1 | grep -E "select|duration" | paste - - | awk '{print $2, $NF}'
