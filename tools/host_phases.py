"""Host time per window of run_windows by phase (perf_counter, no profiler):
counts + schedule, prepare issue, sampler issue, chain issue, and the wall
time per window.  Usage: FGL_HOST_TRACE=2 python tools/host_phases.py [config]"""
import os
import sys
import time
from pathlib import Path
os.environ["FGL_HOST_TRACE"] = "2"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2409_14939_b200 import trainer

name = sys.argv[1] if len(sys.argv) > 1 else "products"
cfg = dict(bench.CONFIGS[name])
dg, feats, labels = bench.build_workload(cfg, "cuda")
wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
mcfg = trainer.ModelConfig(layer_dims=cfg["dims"], fanouts=cfg["fanouts"], arch=cfg["arch"], batch_size=cfg["bs"],
                           window_n=cfg["window"], lr=0.1, seed=0)
pipe = trainer.Pipeline(dg, feats, labels, mcfg, trainer.PipelineFlags(), device="cuda", direct_x0=True)
for _ in pipe.run_windows(wins[:4]):
    pass
torch.cuda.synchronize()
trainer.HOST_TIMES.clear()
K = 30
t0 = time.perf_counter()
for _ in pipe.run_windows(wins[4:4 + K]):
    pass
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"wall per window {(t2 - t0) / K * 1e3:.3f} ms (host loop {(t1 - t0) / K * 1e3:.3f} ms)")
tot = 0.0
for k, v in trainer.HOST_TIMES.items():
    tot += v
    print(f"  {k:22s} {v / K * 1e3:7.3f} ms / window")
print(f"  {'sum':22s} {tot / K * 1e3:7.3f} ms / window")
