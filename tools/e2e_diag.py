"""Diagnose the gap between bench.py's device-timed `value` and its wall-clock
`e2e`: the same windows timed both ways, with and without the per-step loss
read-back, plus the host time spent inside each run_windows iteration."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2409_14939_b200 import trainer  # noqa: E402


def main():
    cfg = dict(bench.CONFIGS["products"])
    dg, feats, labels = bench.build_workload(cfg, "cuda:0")
    wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
    mcfg = trainer.ModelConfig(layer_dims=cfg["dims"], fanouts=cfg["fanouts"], arch="gcn", batch_size=cfg["bs"],
                               window_n=cfg["window"], lr=0.1, seed=0)
    pipe = trainer.Pipeline(dg, feats, labels, mcfg, trainer.PipelineFlags(), device="cuda:0", direct_x0=True)
    K = 40
    it = [0]

    def take(n):
        out = [wins[(it[0] + k) % len(wins)] for k in range(n)]
        it[0] += n
        return out
    from paper_2409_14939_b200 import _lib
    out3 = np.zeros(3, np.int64)
    for _ in pipe.run_windows(take(5)):
        pass
    torch.cuda.synchronize()
    for rep in range(4):
        if rep == 2:
            st = bench.stage_profile(pipe, take(4), cfg, torch)
            print("stage_profile window ms", st["ms"]["window"], flush=True)
        if rep == 3:
            from paper_2409_14939_b200 import _lib
            out3 = np.zeros(3, np.int64)
            _lib.call("fgl_capture_stats", out3.ctypes.data)
            print("capture stats (launches, updates, instantiations)", out3.tolist(), flush=True)
        for mode in ("plain", "copy", "pinned_copy"):
            ws = take(K)
            if mode == "pinned_copy":
                ws = [([torch.from_numpy(s).pin_memory().numpy() for s in seeds], rs) for seeds, rs in ws]
            host_l = [torch.empty(8, dtype=torch.float64).pin_memory() for _ in range(K)]
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            per_it = []
            ti = time.perf_counter()
            for k, (order, losses) in enumerate(pipe.run_windows(ws)):
                if mode != "plain":
                    host_l[k].copy_(losses, non_blocking=True)
                tn = time.perf_counter()
                per_it.append(tn - ti)
                ti = tn
            e1.record()
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            dev = e0.elapsed_time(e1) / 1e3
            pi = np.array(per_it) * 1e3
            print(f"rep {rep} {mode:12s} device {dev / K * 1e3:.3f} ms/win  wall {wall / K * 1e3:.3f} ms/win  "
                  f"host per-iter ms: first {pi[0]:.2f} median {np.median(pi):.3f} max {pi.max():.2f}", flush=True)
            _lib.call("fgl_capture_stats", out3.ctypes.data)
            print("   capture stats (launches, updates, instantiations)", out3.tolist(), flush=True)




def bench_e2e():
    """bench.py's own e2e_measure, repeated."""
    cfg = dict(bench.CONFIGS["products"])
    dg, feats, labels = bench.build_workload(cfg, "cuda:0")
    wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
    mcfg = trainer.ModelConfig(layer_dims=cfg["dims"], fanouts=cfg["fanouts"], arch="gcn", batch_size=cfg["bs"],
                               window_n=cfg["window"], lr=0.1, seed=0)
    pipe = trainer.Pipeline(dg, feats, labels, mcfg, trainer.PipelineFlags(), device="cuda:0", direct_x0=True)
    for _ in pipe.run_windows(wins[:5]):
        pass
    for rep in range(4):
        r = bench.e2e_measure(pipe, wins[5 + 40 * rep: 45 + 40 * rep], torch, 1, "cuda:0")
        print("bench.e2e_measure", r["value"] / 1e9, "G", 6.4e6 / r["value"] * 1e3, "ms/win (approx)", flush=True)


if __name__ == "__main__":
    bench_e2e() if "e2e" in sys.argv else main()
