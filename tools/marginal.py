"""Marginal cost of each stream's work on the pipelined window (products
GCN): run the headline pipeline with one piece of work issued twice (the copy's
results discarded) and report the window time against the baseline.  A
marginal cost near the work's standalone time means the window is throughput
bound on it; near zero means it hides under the critical chain.
  sample2: a second window sampler run on the sampling stream per window
  agg2:    the layer-0 aggregations issued twice on the prepare stream
  chain2:  every tensor-core dense forward issued twice on the chain"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2409_14939_b200 import trainer  # noqa: E402


def run(mode, K=40):
    cfg = dict(bench.CONFIGS["products"])
    dg, feats, labels = bench.build_workload(cfg, "cuda:0")
    wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
    mcfg = trainer.ModelConfig(layer_dims=cfg["dims"], fanouts=cfg["fanouts"], arch="gcn", batch_size=cfg["bs"],
                               window_n=cfg["window"], lr=0.1, seed=0)
    pipe = trainer.Pipeline(dg, feats, labels, mcfg, trainer.PipelineFlags(), device="cuda:0", direct_x0=True)
    P = trainer.Pipeline
    if mode == "sample2":
        orig = P._sample_async

        def twice(self, seed_lists, rng_seeds, slot):
            win = orig(self, seed_lists, rng_seeds, slot)
            if not hasattr(self, "_dup"):
                from paper_2409_14939_b200.sampler import WindowSampler
                self._dup = WindowSampler(self.dg, self.cfg.fanouts, self.cfg.batch_size, self.cfg.window_n,
                                          device=self.device)
            with torch.cuda.stream(self._side):
                nb, off = self._dup.stage(seed_lists, rng_seeds)
                self._dup.run(nb, off, stream=self._side)
            return win
        P._sample_async = twice
    elif mode == "nosample":  # diagnostic: windows re-used, no sampling after the first ones
        orig = P._sample_async
        cache = {}

        def reuse(self, seed_lists, rng_seeds, slot):
            if slot not in cache:
                cache[slot] = orig(self, seed_lists, rng_seeds, slot)
            return cache[slot]
        P._sample_async = reuse
    elif mode == "skip_aggT1":  # diagnostic: drop the transposed layer-1 aggregation (n > 50K rows)
        orig_call = P._call
        state = {}

        def call(self, name, *args):
            if name == "fgl_spmm" and state.get("armed") and int(args[3]) > 50000:
                return 0
            return orig_call(self, name, *args)
        P._call = call
        P._armed_state = state
    elif mode.startswith("skip:"):  # diagnostic: drop the named library calls (results invalid)
        names = set(mode[5:].split(","))
        orig_call = P._call
        state = {"n": 0}

        def call(self, name, *args):
            if name in names and state.get("armed"):
                return 0
            return orig_call(self, name, *args)
        P._call = call
        P._armed_state = state
    elif mode in ("agg2", "chain2"):
        orig_call = P._call
        target = "fgl_spmm_gather" if mode == "agg2" else "fgl_dense_fwd"

        def call(self, name, *args):
            rc = orig_call(self, name, *args)
            if name == target:
                orig_call(self, name, *args)
            return rc
        P._call = call
    for _ in pipe.run_windows(wins[:5]):
        pass
    torch.cuda.synchronize()
    if hasattr(P, "_armed_state"):
        P._armed_state["armed"] = True
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in pipe.run_windows(wins[5:5 + K]):
        pass
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "base"
    print(f"{mode:8s} {run(mode):.3f} ms/window", flush=True)
