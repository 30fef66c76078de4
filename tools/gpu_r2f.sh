#!/bin/bash
# Round-2 evidence run: gradient parity re-check, ncu captures of the stage
# kernels (traffic + source), a launch list, the config-5 GIN batch sweep and
# products at the paper's batch 8000.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_configs.py -q -k batch_gradients > $O/grad_test.log 2>&1
bash tools/ncu_evidence.sh $1 > $O/ncu_evidence.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches.csv python bench.py --profile --no-cpu-baseline > $O/launches.log 2>&1
for bs in 512 1024 2048 4096 8192; do
  timeout 600 python bench.py --config gin --bs $bs --steps 10 --warmup 3 --no-cpu-baseline > $O/gin_bs$bs.json 2> $O/gin_bs$bs.err
done
timeout 600 python bench.py --bs 8000 --steps 10 --warmup 3 --no-cpu-baseline > $O/products_bs8000.json 2> $O/products_bs8000.err
