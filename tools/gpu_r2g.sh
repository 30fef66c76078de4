#!/bin/bash
# select v2 + spmm_pipe register-bound A/B: parity tests, stage microbenchmarks, bench lines.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_scale.py tests/test_gpu_configs.py tests/test_gpu_spmm_gather.py -q -x > $O/test.log 2>&1
for v in 1 2; do FGL_SELV=$v timeout 300 python tools/bench_stages.py --windows 20 > $O/stages_selv$v.json 2>&1; done
for m in 4 5; do FGL_PIPE_MINB=$m timeout 300 python tools/spmm_gather_bench.py > $O/spmm_minb$m.txt 2>&1; done
for v in 1 2; do FGL_SELV=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_selv$v.json 2> $O/bench_selv$v.err; done
