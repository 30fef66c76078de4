"""Which resource binds the pipelined window?  Re-time run_windows with
selected compute entry points turned into no-ops (results become garbage;
sampling and all sizes are unaffected) and report wall / host-blocked /
host-issue time per window.  Usage: sensitivity.py [fn,fn,...] (C-ABI names)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2409_14939_b200 import trainer, sampler as S

skip = set(sys.argv[1].split(",")) if len(sys.argv) > 1 and sys.argv[1] else set()
cfg = bench.CONFIGS["products"]
dg, feats, labels = bench.build_workload(cfg, "cuda")
wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
mcfg = trainer.ModelConfig(layer_dims=cfg["dims"], fanouts=cfg["fanouts"], arch="gcn", batch_size=1024, window_n=8,
                           lr=0.1, seed=0)
pipe = trainer.Pipeline(dg, feats, labels, mcfg, trainer.PipelineFlags(), device="cuda", direct_x0=True)
orig_call = trainer.Pipeline._call
def call(self, name, *args):
    if name in skip:
        return
    return orig_call(self, name, *args)
trainer.Pipeline._call = call
blocked = [0.0]
orig = S.DeviceWindow.host_counts
def timed(self):
    t = time.perf_counter(); r = orig(self); blocked[0] += time.perf_counter() - t; return r
S.DeviceWindow.host_counts = timed
orig_sched = trainer.Pipeline.schedule
def tsched(self, win, nb):
    t = time.perf_counter(); r = orig_sched(self, win, nb); blocked[0] += time.perf_counter() - t; return r
trainer.Pipeline.schedule = tsched
for _ in pipe.run_windows(wins[:3]): pass
torch.cuda.synchronize()
blocked[0] = 0.0
K = 30
t0 = time.perf_counter()
for _ in pipe.run_windows(wins[3:3 + K]): pass
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / K * 1e3
import ctypes
from paper_2409_14939_b200 import _lib as _L
st3 = (ctypes.c_int64 * 3)()
_L.call("fgl_capture_stats", ctypes.cast(st3, ctypes.c_void_p))
print(f"graphs: launches {st3[0]} updates {st3[1]} instantiations {st3[2]}, eager fallbacks {pipe.graph_fallbacks}")
print(f"skip={sorted(skip)}: wall {tot:.3f} ms/window, host blocked {blocked[0] / K * 1e3:.3f}, "
      f"issuing {tot - blocked[0] / K * 1e3:.3f}", flush=True)
