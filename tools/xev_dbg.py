import sys; sys.path.insert(0,'.')
import torch, bench
from paper_2409_14939_b200 import trainer
cfg = bench.CONFIGS["products"]
dg, feats, labels = bench.build_workload(cfg, "cuda")
wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
m = trainer.ModelConfig(layer_dims=cfg["dims"], fanouts=cfg["fanouts"], arch="gcn", batch_size=1024, window_n=8, lr=0.1, seed=0)
pipe = trainer.Pipeline(dg, feats, labels, m, trainer.PipelineFlags(), device="cuda", direct_x0=True)
orig = trainer.Pipeline._graphed
def g(self, stream, slot, fn):
    import traceback
    try:
        return orig(self, stream, slot, fn)
    finally:
        pass
for _ in pipe.run_windows(wins[:6]): pass
torch.cuda.synchronize()
print("graph fallbacks", pipe.graph_fallbacks)
