"""Per-hop split of a products window's Philox draws: frontier entries and
draws by degree class (hubs d > 2048 go to select_hub_kernel), to size the
select kernels' work."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2409_14939_b200 import sampler as S  # noqa: E402

cfg = bench.CONFIGS["products"]
dg, feats, labels = bench.build_workload(cfg, "cuda")
wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
ws = S.WindowSampler(dg, cfg["fanouts"], cfg["bs"], cfg["window"])
win = ws.sample(*wins[3])
off = dg.row_offsets
for h in range(len(cfg["fanouts"])):
    f = win.frontier(h).long()
    d = (off[f + 1] - off[f]).cpu().numpy()
    tot = d.sum()
    print(f"hop {h} fan {cfg['fanouts'][h]}: frontier {len(d)}, draws {tot / 1e6:.2f}M, mean deg {d.mean():.1f}")
    for lo, hi in [(0, 16), (16, 64), (64, 256), (256, 2048), (2048, 1 << 40)]:
        m = (d > lo) & (d <= hi)
        print(f"   deg ({lo},{hi}]: nodes {m.sum():7d} ({m.mean() * 100:5.1f}%)  draws {d[m].sum() / 1e6:6.2f}M "
              f"({d[m].sum() / tot * 100:5.1f}%)")
