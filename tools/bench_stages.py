"""Stage microbenchmarks on the products-shaped workload (device time, CUDA
events): the window sampler alone, and one full window split by stage.
Usage: python tools/bench_stages.py [--windows 20]"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_14939_b200 import sampler as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--windows", type=int, default=20)
    ap.add_argument("--config", default="products")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    dg, feats, labels = bench.build_workload(cfg, "cuda")
    wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
    ws = S.WindowSampler(dg, cfg["fanouts"], cfg["bs"], cfg["window"])
    for k in range(3):
        ws.sample(*wins[k]).host_counts()
    staged = []
    for k in range(args.windows):
        staged.append(ws.stage(*wins[3 + k]))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot_ms, edges, draws, fronts = 0.0, 0, 0, [0] * len(cfg["fanouts"])
    for k in range(args.windows):
        nb, off = ws.stage(*wins[3 + k])
        e0.record()
        win = ws.run(nb, off)
        e1.record()
        torch.cuda.synchronize()
        tot_ms += e0.elapsed_time(e1)
        edges += win.total_edges()
        draws += sum(win.draws(b) for b in range(nb))
        for h in range(len(fronts)):
            fronts[h] += win.front_total(h)
    print(json.dumps({"sampler_ms_per_window": tot_ms / args.windows,
                      "edges_per_window": edges / args.windows,
                      "draws_per_window": draws / args.windows,
                      "frontier_per_hop_per_window": [f / args.windows for f in fronts],
                      "unique_per_window": win.unique_total(),
                      "draws_per_s": draws / (tot_ms / 1e3)}))


if __name__ == "__main__":
    main()
