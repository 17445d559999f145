"""Print the last N launches of an ncu launch list (duration, DRAM bytes) in
launch order: the per-kernel anatomy of one decode layer."""
import csv
import sys

path, last = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12
rows = list(csv.reader(open(path)))
hdr, seq = None, {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        e = seq.setdefault(int(d["ID"]), {"name": d["Kernel Name"], "grid": d.get("Grid Size", "")})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
ids = sorted(seq)[-last:]
tot = 0.0
for i in ids:
    e = seq[i]
    t = e.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    b = (e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)) / 1e6
    print(f"{e['name'][:60]:60s} {e['grid']:>14s} {t:8.2f}us {b:8.2f}MB {b / max(t, 1e-9) / 1e3 * 1e3:7.1f}GB/s")
print(f"total {tot:.2f} us")
