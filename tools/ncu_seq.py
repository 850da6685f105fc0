"""Print an ncu --csv launch list (gpu__time_duration.sum) in launch order.

python tools/ncu_seq.py launches.csv [first] [count]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
out = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v = v / 1e3 if u in ("nsecond", "ns") else (v * 1e3 if u in ("msecond", "ms") else v)
        g = d.get("Grid Size", "")
        out.append((d["ID"], d["Kernel Name"][:70], g, v))
a = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else len(out)
for i, (kid, name, g, v) in enumerate(out[a:a + n]):
    print(f"{a + i:5d} {v:9.1f}us  {g:>16s}  {name}")
