"""Live device time of each call of the weight-dependent chain (main stream,
eager launches, FGL_GRAPH=0) while sampling / prepare / layer-0 aggregation
run on their streams: CUDA events around every Pipeline._call made from
batch_step.  Gaps between calls (waits, launch latency) are reported too."""
import os, sys, collections
from pathlib import Path
os.environ["FGL_GRAPH"] = "0"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2409_14939_b200 import trainer

cfg = bench.CONFIGS["products"]
dg, feats, labels = bench.build_workload(cfg, "cuda")
wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
mcfg = trainer.ModelConfig(layer_dims=cfg["dims"], fanouts=cfg["fanouts"], arch="gcn", batch_size=1024, window_n=8,
                           lr=0.1, seed=0)
pipe = trainer.Pipeline(dg, feats, labels, mcfg, trainer.PipelineFlags(), device="cuda", direct_x0=True)
for _ in pipe.run_windows(wins[:3]): pass
torch.cuda.synchronize()
rec = []
orig_call = trainer.Pipeline._call
in_step = [False]
def call(self, name, *args):
    if not in_step[0]:
        return orig_call(self, name, *args)
    cur = self._cur()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cur)
    orig_call(self, name, *args)
    b.record(cur)
    rec.append((name, a, b))
trainer.Pipeline._call = call
orig_step = trainer.Pipeline._batch_step_body
def step(self, *a, **k):
    in_step[0] = True
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(self._cur())
    try:
        return orig_step(self, *a, **k)
    finally:
        in_step[0] = False
        s1.record(self._cur())
        rec.append(("<batch_step total>", s0, s1))
trainer.Pipeline._batch_step_body = step
K = 10
for _ in pipe.run_windows(wins[3:3 + K]): pass
torch.cuda.synchronize()
acc = collections.defaultdict(lambda: [0, 0.0])
for name, a, b in rec:
    acc[name][0] += 1
    acc[name][1] += a.elapsed_time(b) * 1e3
nb = K * 8
print(f"per batch (live, {nb} batches):")
for k, (c, t) in sorted(acc.items(), key=lambda x: -x[1][1]):
    print(f"  {k:28s} {c / nb:5.1f} calls  {t / nb:8.1f} us")
