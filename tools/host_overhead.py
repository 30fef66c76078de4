"""Host-side issue time of one window's prepare + 8 batch steps (no syncs
inside), vs the device time of the same work: is the host the limiter?"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
from paper_2409_14939_b200 import trainer

cfg = bench.CONFIGS["products"]
dg, feats, labels = bench.build_workload(cfg, "cuda")
wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
mcfg = trainer.ModelConfig(layer_dims=cfg["dims"], fanouts=cfg["fanouts"], arch=cfg["arch"], batch_size=cfg["bs"],
                           window_n=cfg["window"], lr=0.1, seed=0)
pipe = trainer.Pipeline(dg, feats, labels, mcfg, trainer.PipelineFlags(), device="cuda", direct_x0=True)
for k in range(3):
    pipe.run_window(*wins[k])
torch.cuda.synchronize()
host, dev = [], []
for k in range(3, 13):
    win = pipe.sampler.sample(*wins[k])
    win.host_counts()
    order = pipe.schedule(win, len(wins[k][0]))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # stall the GPU so the host issue time is visible on its own
    torch.cuda._sleep(50_000_000)
    t0 = time.perf_counter()
    e0.record()
    layers = pipe.prepare(win)
    for j, b in enumerate(order):
        pipe.batch_step(win, b, order[j - 1] if j else None, j, layers, j % 2)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    host.append((t1 - t0) * 1e3)
    dev.append(e0.elapsed_time(e1))
print(f"host issue ms/window: {np.median(host):.3f}   device ms (prepare+compute): {np.median(dev):.3f}   launches/window: {pipe.gpu_launches}")
