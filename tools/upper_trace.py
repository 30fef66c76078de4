import os, sys, ctypes
os.environ["FGL_UPDBG"] = "1"
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
from paper_2409_14939_b200 import trainer, _lib
cfg = bench.CONFIGS["products"]
dg, feats, labels = bench.build_workload(cfg, "cuda")
wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
mcfg = trainer.ModelConfig(layer_dims=cfg["dims"], fanouts=cfg["fanouts"], arch="gcn", batch_size=1024, window_n=8, lr=0.1, seed=0)
pipe = trainer.Pipeline(dg, feats, labels, mcfg, trainer.PipelineFlags(), device="cuda", direct_x0=True)
for k in range(3):
    pipe.run_window(*wins[k])
torch.cuda.synchronize()
buf = np.zeros(64, dtype=np.int64)
_lib.lib().fgl_debug_upper_trace(buf.ctypes.data_as(ctypes.c_void_p))
t = buf[buf > 0]
names = ["L1 agg", "L1 dense", "L2 agg", "L2 dense", "loss", "L2 wgrad+dgrad", "L2->L1 agg", "L1 wgrad+dgrad", "reduce"]
d = np.diff(t) / 1e3
for i, x in enumerate(d):
    print(f"{names[i] if i < len(names) else i}: {x:.2f} us")
print("total", (t[-1] - t[0]) / 1e3)
