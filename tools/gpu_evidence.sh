#!/bin/bash
# Round-2 timeline / throughput evidence: live + serialised CUPTI timelines,
# marginal-cost runs, the sampler's per-kernel split and the Philox
# occupancy probe.  Usage: tools/gpu_evidence.sh <tag>
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/$1; mkdir -p $O
python tools/timeline.py $O/tl_live.json > /dev/null 2>&1
FGL_GRAPH=0 CUDA_LAUNCH_BLOCKING=1 python tools/timeline.py $O/tl_serial.json > /dev/null 2>&1
for m in base sample2 agg2 chain2; do python tools/marginal.py $m 2>/dev/null; done > $O/marginal.txt
python tools/sampler_tl.py 2>&1 | grep -v -i warn > $O/sampler_tl.txt
(cd tools/probes && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2409_14939_b200/csrc -o philox_occ philox_occ.cu ../../paper_2409_14939_b200/build/abi.o -lcuda 2>/dev/null; ./philox_occ) > $O/philox_occ.txt 2>&1
