#!/bin/bash
# Full GPU check of the committed state: every -m gpu test, smoke(), the default
# bench line and the per-config bench lines.  Usage: tools/gpu_check.sh <tag>
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $O/test.log 2>&1; echo "pytest rc=$?" >> $O/test.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
