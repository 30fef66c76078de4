"""Per-batch critical path of a tools/timeline.py capture: the chain stream's
and the per-batch side streams' kernels between consecutive SGD launches, with
start offsets, durations and idle gaps (what the batch waited on).
Usage: python tools/chain_path.py TL.json [batches]"""
import json
import re
import sys


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("void ", "").replace("fgl::", "")
    return re.sub(r"\(.*", "", n)[:34]


ev = json.load(open(sys.argv[1]))
ev.sort(key=lambda e: e["ts"])
nshow = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sgd = [e for e in ev if "sgd" in e["name"]]
chain_stream = sgd[0]["stream"]
side = {e["stream"] for e in ev if e["stream"] not in (13, 17, 21, chain_stream)}
per = []
tot = {}
for i in range(1, len(sgd)):
    t0, t1 = sgd[i - 1]["ts"] + sgd[i - 1]["dur"], sgd[i]["ts"] + sgd[i]["dur"]
    ks = [e for e in ev if (e["stream"] == chain_stream or e["stream"] in side) and t0 <= e["ts"] < t1]
    per.append(t1 - t0)
    for e in ks:
        tot.setdefault(short(e["name"]), []).append(e["dur"])
    if i <= nshow:
        print(f"batch {i}: {t1 - t0:.1f} us")
        for e in ks:
            tag = "chain" if e["stream"] == chain_stream else "side "
            print(f"   {tag} +{e['ts'] - t0:7.1f}  {e['dur']:6.1f}  {short(e['name'])}")
per.sort()
print(f"batches {len(per)}: median {per[len(per) // 2]:.1f} us, mean {sum(per) / len(per):.1f} us, max {per[-1]:.1f}")
for k, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
    print(f"   {k:36s} n {len(v):3d}  avg {sum(v) / len(v):6.1f} us")
