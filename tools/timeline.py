"""Kernel timeline of the headline pipeline (products GCN, CUDA graphs, all
streams live) from CUPTI via torch.profiler: every kernel's start / end and
stream over a few windows, written as JSON for offline analysis
(tools/timeline_report.py).  Usage: python tools/timeline.py OUT.json [config]"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2409_14939_b200 import trainer  # noqa: E402


def main():
    out = sys.argv[1]
    name = sys.argv[2] if len(sys.argv) > 2 else "products"
    cfg = dict(bench.CONFIGS[name])
    dg, feats, labels = bench.build_workload(cfg, "cuda:0")
    wins, _ = bench.epoch_windows(dg.num_nodes, cfg)
    mcfg = trainer.ModelConfig(layer_dims=cfg["dims"], fanouts=cfg["fanouts"], arch=cfg["arch"],
                               batch_size=cfg["bs"], window_n=cfg["window"], lr=0.1, seed=0)
    pipe = trainer.Pipeline(dg, feats, labels, mcfg, trainer.PipelineFlags(), device="cuda:0", direct_x0=True)
    for _ in pipe.run_windows(wins[:6]):
        pass
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    acts = [ProfilerActivity.CUDA] + ([ProfilerActivity.CPU] if os.environ.get("FGL_HOST_TRACE") == "1" else [])
    with profile(activities=acts) as prof:
        for _ in pipe.run_windows(wins[6:16]):
            pass
        torch.cuda.synchronize()
    prof.export_chrome_trace(out + ".trace.json")
    tr = json.load(open(out + ".trace.json"))
    def launch_args(a):
        return {k: a.get(k) for k in ("grid", "block", "registers per thread", "shared memory",
                                      "est. achieved occupancy %", "warps per SM", "blocks per SM") if k in a}
    ev = [dict(name=e["name"], ts=e["ts"], dur=e["dur"], stream=e.get("args", {}).get("stream"),
               cat=e.get("cat"), **launch_args(e.get("args", {}))) for e in tr["traceEvents"]
          if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    ev += [dict(name=e["name"], ts=e["ts"], dur=e["dur"], stream="host", cat="host") for e in tr["traceEvents"]
           if e.get("ph") == "X" and e.get("cat") == "user_annotation" and e["name"].startswith("window")]
    json.dump(ev, open(out, "w"))
    Path(out + ".trace.json").unlink()
    print("events", len(ev))


if __name__ == "__main__":
    main()
