"""Per-kernel DRAM bytes and durations over one profiled bench window (ncu
--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--cache-control none CSV): total bytes per window vs the step time says
whether the pipeline as a whole is HBM bound."""
import collections, csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mi, ui, ni, idi = (h.index(x) for x in ('Kernel Name', 'Metric Value', 'Metric Unit', 'Metric Name', 'ID'))
scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'nsecond': 1e-3, 'usecond': 1, 'msecond': 1e3, 'ns': 1e-3, 'us': 1}
per = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    name = re.sub(r'^void ', '', r[ki].replace('(anonymous namespace)::', '')).split('(')[0]
    per[r[idi]]['name'] = name
    per[r[idi]][r[ni]] = float(r[mi].replace(',', '')) * scale.get(r[ui], 1.0)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for v in per.values():
    a = agg[v['name']]
    a[0] += 1
    a[1] += v.get('dram__bytes_read.sum', 0) + v.get('dram__bytes_write.sum', 0)
    a[2] += v.get('gpu__time_duration.sum', 0)
tb = sum(a[1] for a in agg.values())
tt = sum(a[2] for a in agg.values())
print(f"launches {sum(a[0] for a in agg.values())}  DRAM bytes {tb / 1e6:.1f} MB  kernel time {tt / 1e3:.2f} ms  "
      f"(avg {tb / tt / 1e3 if tt else 0:.0f} GB/s while a kernel runs)")
for k, (c, b, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{k[:60]:60s} {c:5d} {b / 1e6:9.1f} MB {t / 1e3:8.3f} ms {b / t / 1e3 if t else 0:7.0f} GB/s")
