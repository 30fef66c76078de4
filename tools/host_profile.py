"""cProfile of the host side of run_windows (products GCN): where the ~2.5 ms
of per-window issue time goes."""
import cProfile, pstats, sys
from pathlib import Path
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
import collections, time
from paper_2409_14939_b200 import _lib
acc = collections.defaultdict(lambda: [0, 0.0])
orig = _lib.call
def timed(name, *a):
    t = time.perf_counter(); orig(name, *a); acc[name][0] += 1; acc[name][1] += time.perf_counter() - t
_lib.call = timed
import paper_2409_14939_b200.sampler as S
S._lib.call = timed
for _ in pipe.run_windows(wins[3:23]): pass
torch.cuda.synchronize()
_lib.call = orig
print("per window, C-ABI calls by host time:")
for k, (c, t) in sorted(acc.items(), key=lambda x: -x[1][1]):
    print(f"  {k:32s} {c / 20:6.1f} calls  {t / 20 * 1e3:7.3f} ms  {t / c * 1e6:6.1f} us/call")
pr = cProfile.Profile()
pr.enable()
for _ in pipe.run_windows(wins[23:43]): pass
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(12)
