"""Top stalled SASS instructions of an `ncu --page source --csv --print-source
sass` export: python tools/sass_top.py file.csv [n]"""
import csv, sys
r = list(csv.reader(open(sys.argv[1])))
h = r[1]
i = h.index("Warp Stall Sampling (All Samples)")
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
rows = [x for x in r[2:] if len(x) > i and x[i].isdigit()]
tot = sum(int(x[i]) for x in rows)
order = sorted(range(len(rows)), key=lambda j: -int(rows[j][i]))
for j in order[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    x = rows[j]
    top = sorted(((int(x[h.index(k)]), k[6:]) for k in stalls), reverse=True)[:3]
    print(f"{int(x[i]) / tot * 100:5.1f}%  #{j:<5d} {x[1].strip()[:60]:60s} {top}")
print("total samples", tot)
