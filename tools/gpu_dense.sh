#!/bin/bash
# dense kernel check + microbench on one GPU
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_dense.py -x -q > $O/dense_test.log 2>&1; echo "rc=$?" >> $O/dense_test.log
for sh in "129000 100 64" "15000 64 64" "1024 64 47"; do
  timeout 120 python tools/dense_bench.py $sh >> $O/dense_bench.log 2>&1
  FGL_DENSE=v2 timeout 120 python tools/dense_bench.py $sh >> $O/dense_bench_v2.log 2>&1
done
tail -5 $O/dense_test.log; cat $O/dense_bench.log $O/dense_bench_v2.log
