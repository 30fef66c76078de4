"""SM-capacity demand of a tools/timeline.py capture: for every kernel, the
fraction of the GPU's per-SM resources (registers, thread slots, shared
memory) its resident CTAs hold while it runs, times its duration; summed per
kernel name and per window.  A total near the window time means the GPU is
capacity-bound (kernels queue for SM resources rather than for a dependency).
Usage: python tools/sm_demand.py TL.json [windows]"""
import collections
import json
import re
import sys


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("void ", "").replace("fgl::", "")
    return re.sub(r"\(.*", "", n)[:40]


ev = [e for e in json.load(open(sys.argv[1])) if e.get("cat") == "kernel" and "grid" in e]
nwin = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
SMS, RF, THR, SMEM, BLK = 148, 65536, 2048, 228 * 1024, 32
acc = collections.defaultdict(lambda: [0.0, 0.0, 0])
for e in ev:
    g = e["grid"][0] * e["grid"][1] * e["grid"][2]
    t = e["block"][0] * e["block"][1] * e["block"][2]
    regs = max(1, e.get("registers per thread") or 1)
    sm = (e.get("shared memory") or 0) + 1024
    w = (t + 31) // 32
    per_sm = min(BLK, THR // t, RF // (((regs * 32 + 255) // 256) * 256 * w), SMEM // sm)
    per_sm = max(per_sm, 1)
    resident = min(g / SMS, per_sm)  # CTAs per SM while it runs (ignores tails)
    frac = max(resident * t / THR, resident * regs * t / RF, resident * sm / SMEM)
    frac = min(frac, 1.0)
    a = acc[short(e["name"])]
    a[0] += e["dur"]
    a[1] += e["dur"] * frac
    a[2] += 1
tot = sum(v[1] for v in acc.values())
print(f"SM-capacity demand {tot / nwin:.1f} us per window (kernel time {sum(v[0] for v in acc.values()) / nwin:.1f} us)")
for k, (d, f, n) in sorted(acc.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {k:40s} n/win {n / nwin:5.1f}  dur {d / nwin:7.1f} us  demand {f / nwin:7.1f} us  ({f / d:4.2f} of the GPU)")
