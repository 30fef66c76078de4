"""Record dram__bytes_read.sum + dram__bytes_write.sum (and duration) of one
ncu --set full capture into profiles/ncu_traffic.json under a kernel key.
Usage: python tools/ncu_traffic.py <report.ncu-rep> <kernel-key> [note]"""
import csv, io, json, subprocess, sys
from pathlib import Path

rep, key = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
def get(k):
    i = h.index(k)
    x = float(v[i].replace(",", ""))
    u = units[i]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "ns": 1e-9}
    return x * scale.get(u, 1)
out = {"dram_read_bytes": get("dram__bytes_read.sum"), "dram_write_bytes": get("dram__bytes_write.sum"),
       "duration_s": get("gpu__time_duration.sum"), "report": Path(rep).name, "note": note}
out["traffic_bytes"] = out["dram_read_bytes"] + out["dram_write_bytes"]
p = Path(__file__).resolve().parents[1] / "profiles" / "ncu_traffic.json"
d = json.loads(p.read_text()) if p.exists() else {}
d[key] = out
p.write_text(json.dumps(d, indent=1) + "\n")
print(key, out)
