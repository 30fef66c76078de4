"""Top source lines of an ncu report by warp-stall samples:
ncu -i X.ncu-rep --page source --csv --print-source cuda,sass | python tools/ncu_src_top.py [N]"""
import csv
import sys

rows = list(csv.reader(sys.stdin))
cur = None
out = []
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 8 or not r[0].isdigit():
        continue
    try:
        s, ins = int(r[4]), int(r[7])
    except ValueError:
        continue
    out.append((s, ins, cur, int(r[0]), r[1][:100]))
tot = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print("total stall samples", tot, "warp instructions", ti)
for s, ins, f, ln, src in sorted(out, reverse=True)[: int(sys.argv[1]) if len(sys.argv) > 1 else 40]:
    print(f"{s / tot * 100:5.1f}%s {ins / ti * 100:5.1f}%i {f}:{ln} {src}")
