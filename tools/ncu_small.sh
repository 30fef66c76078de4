#!/bin/bash
# ncu --set full of the sampler's latency-bound launches (products window).
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
N="ncu --set full --clock-control none --import-source on --profile-from-start off"
B="python bench.py --profile --no-cpu-baseline"
timeout 600 $N -k regex:select_bal2 -s 0 -c 1 -o $O/sel_hop0 $B > $O/a.log 2>&1
timeout 600 $N -k regex:bm_compact -s 4 -c 1 -o $O/compact_uniq $B > $O/b.log 2>&1
timeout 600 $N -k regex:translate_kernel -s 2 -c 1 -o $O/translate_h2 $B > $O/c.log 2>&1
