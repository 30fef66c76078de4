"""Per-kernel device time of the window sampler alone (products graph, 8 x 1024
seeds), CUPTI via torch.profiler, eager launches on one stream: which of the
~35 sampler launches per window cost what.  Usage: python tools/sampler_tl.py [config]"""
import collections
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2409_14939_b200 import sampler as S  # noqa: E402


def main():
    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "products"]
    dg, feats, labels = bench.build_workload(cfg, "cuda")
    wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
    ws = S.WindowSampler(dg, cfg["fanouts"], cfg["bs"], cfg["window"])
    for k in range(3):
        ws.sample(*wins[k]).host_counts()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    nw = 10
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for k in range(nw):
            nb, off = ws.stage(*wins[3 + k])
            ws.run(nb, off)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    seq = collections.OrderedDict()
    for e in evs:
        n = e.name.replace("fgl::(anonymous namespace)::", "").replace("fgl::", "").split("(")[0][:40]
        seq.setdefault(n, []).append(e.device_time)
    tot = sum(sum(v) for v in seq.values()) / nw
    print(f"sampler kernels: {tot:.1f} us per window (sum of device times)")
    for n, v in sorted(seq.items(), key=lambda x: -sum(x[1])):
        per = len(v) / nw
        print(f"  {n:40s} {per:4.1f}/win  {sum(v) / nw:8.1f} us/win   per launch: "
              + " ".join(f"{x:.1f}" for x in v[: int(per)]))


if __name__ == "__main__":
    main()
