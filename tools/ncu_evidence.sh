#!/bin/bash
# One ncu --set full capture per hot kernel of the bench's profiled window
# (products GCN; host-store config for the gather) -> gpurun_out/$1/*.ncu-rep
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
N="ncu --set full --clock-control none --import-source on --profile-from-start off"
B="python bench.py --profile --no-cpu-baseline"
timeout 600 $N -k regex:select_bal2 -s 2 -c 1 -o $O/select_bal2 $B > $O/l1.log 2>&1
timeout 600 $N -k regex:spmm_lean_kernel -s 0 -c 1 -o $O/spmm_l0 $B > $O/l2.log 2>&1
timeout 600 $N -k regex:tc_dense4_kernel -s 0 -c 1 -o $O/dense4_l0 $B > $O/l3.log 2>&1
timeout 600 $N -k regex:tc_dense4_kernel -s 2 -c 1 -o $O/dense4_dgrad $B > $O/l3b.log 2>&1
timeout 600 $N -k regex:tc_wgrad3_kernel -s 1 -c 1 -o $O/wgrad_l0 $B > $O/l4.log 2>&1
if [ -n "$2" ]; then
timeout 900 $N -k regex:gather_rows -s 1 -c 1 -o $O/gather_host $B --config products_host > $O/l5.log 2>&1
fi
ls -la $O
