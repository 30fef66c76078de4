"""Summarise a tools/timeline.py capture: per-stream busy time, per-kernel
totals, GPU idle time, and the critical (chain) stream's per-batch split."""
import collections
import json
import re
import sys


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("void ", "").replace("fgl::", "")
    n = re.sub(r"\(.*", "", n)
    return n[:48]


def main():
    ev = json.load(open(sys.argv[1]))
    ev.sort(key=lambda e: e["ts"])
    t0 = ev[0]["ts"]
    t1 = max(e["ts"] + e["dur"] for e in ev)
    span = t1 - t0
    print(f"span {span / 1e3:.3f} ms, {len(ev)} events")
    # union of busy intervals (any kernel running)
    busy = 0.0
    cur_s, cur_e = None, None
    for e in ev:
        s, en = e["ts"], e["ts"] + e["dur"]
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, en
        else:
            cur_e = max(cur_e, en)
    busy += cur_e - cur_s
    print(f"GPU busy (any kernel) {busy / span * 100:.1f}% of span")
    by_stream = collections.defaultdict(list)
    for e in ev:
        by_stream[e["stream"]].append(e)
    print("\nper stream: kernels, summed dur (ms), span share")
    for st, es in sorted(by_stream.items(), key=lambda x: -sum(e["dur"] for e in x[1])):
        d = sum(e["dur"] for e in es)
        print(f"  stream {st}: {len(es):5d} ev  {d / 1e3:8.3f} ms  {d / span * 100:5.1f}%")
        k = collections.defaultdict(lambda: [0, 0.0])
        for e in es:
            k[short(e["name"])][0] += 1
            k[short(e["name"])][1] += e["dur"]
        for n, (c, t) in sorted(k.items(), key=lambda x: -x[1][1])[:12]:
            print(f"      {n:50s} {c:5d}  {t / 1e3:8.3f} ms  avg {t / c:7.1f} us")
    # chain stream = the one with the sgd kernel
    chain = None
    for st, es in by_stream.items():
        if any("sgd" in e["name"] for e in es):
            chain = st
    if chain is not None:
        es = by_stream[chain]
        gaps = [es[i + 1]["ts"] - (es[i]["ts"] + es[i]["dur"]) for i in range(len(es) - 1)]
        gap_total = sum(g for g in gaps if g > 0)
        cspan = es[-1]["ts"] + es[-1]["dur"] - es[0]["ts"]
        print(f"\nchain stream {chain}: span {cspan / 1e3:.3f} ms, kernels {sum(e['dur'] for e in es) / 1e3:.3f} ms, "
              f"gaps {gap_total / 1e3:.3f} ms over {len(gaps)} boundaries")
        big = sorted(((g, short(es[i]['name']), short(es[i + 1]['name'])) for i, g in enumerate(gaps)), reverse=True)[:10]
        for g, a, b in big:
            print(f"    gap {g:7.1f} us after {a} before {b}")
        # who runs while the chain waits: kernels overlapping chain gaps > 5 us
        occ = collections.defaultdict(float)
        gsum = 0.0
        others = [e for e in ev if e["stream"] != chain]
        for i in range(len(es) - 1):
            g0, g1 = es[i]["ts"] + es[i]["dur"], es[i + 1]["ts"]
            if g1 - g0 < 5:
                continue
            gsum += g1 - g0
            for e in others:
                o = min(g1, e["ts"] + e["dur"]) - max(g0, e["ts"])
                if o > 0:
                    occ[short(e["name"])] += o
        print(f"\nkernels overlapping chain gaps > 5 us (total gap {gsum / 1e3:.3f} ms):")
        for n, t in sorted(occ.items(), key=lambda x: -x[1])[:15]:
            print(f"    {n:50s} {t / 1e3:8.3f} ms")
        # sequence of one batch (between consecutive sgd kernels)
        idx = [i for i, e in enumerate(es) if "sgd" in e["name"]]
        if len(idx) > 3:
            i0, i1 = idx[len(idx) // 2], idx[len(idx) // 2 + 1]
            print("\none batch on the chain stream (kernel, dur us, gap before us):")
            for i in range(i0 + 1, i1 + 1):
                print(f"    {short(es[i]['name']):50s} {es[i]['dur']:7.1f}  {es[i]['ts'] - es[i - 1]['ts'] - es[i - 1]['dur']:6.1f}")


if __name__ == "__main__":
    main()
