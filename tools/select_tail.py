"""Per-warp finish-time distribution of the last select_bal launch (FGL_SELDBG)."""
import os, sys, ctypes
os.environ["FGL_SELDBG"] = "1"
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
from paper_2409_14939_b200 import sampler as S, _lib
cfg = bench.CONFIGS["products"]
dg, feats, labels = bench.build_workload(cfg, "cuda")
wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
ws = S.WindowSampler(dg, cfg["fanouts"], cfg["bs"], cfg["window"])
for k in range(4):
    ws.sample(*wins[k]).host_counts()
torch.cuda.synchronize()
buf = np.zeros(4096, dtype=np.int64)
_lib.lib().fgl_debug_select_finish(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(4096))
t0 = buf[0]
f = np.sort(buf[1:][buf[1:] > 0] - t0) / 1e3
print("warps", len(f), "finish us: p10 %.1f p50 %.1f p90 %.1f p99 %.1f max %.1f" % tuple(np.percentile(f, [10, 50, 90, 99, 100])))
