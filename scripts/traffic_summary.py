"""Combine ncu DRAM launch lists of scripts/traffic_attn.py runs with their
algorithmic byte counts -> profiles/rN/traffic_decode_attn.json (read by
bench.py for roofline.traffic).

    python scripts/traffic_summary.py OUT.json A.csv A.json [B.csv B.json ...]"""
import csv
import json
import sys


def dram_total(path):
    rows = list(csv.reader(open(path)))
    hdr, tot, ids = None, 0.0, set()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if "decode_attn" in d["Kernel Name"] and d["Metric Name"].startswith("dram__bytes"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d.get("Metric Unit", "byte"), 1)
                tot += float(d["Metric Value"].replace(",", "")) * scale
                ids.add(d["ID"])
    return tot, len(ids)


out, args = sys.argv[1], sys.argv[2:]
src = None
if args and args[0].startswith("--source="):
    src, args = args[0][len("--source="):], args[1:]
caps, D, A, N = [], 0.0, 0.0, 0
for c, j in zip(args[::2], args[1::2]):
    dram, n = dram_total(c)
    acc = json.loads([x for x in open(j) if x.startswith("{")][0])
    assert n == acc["launches"], (c, n, acc["launches"])
    caps.append({"B": acc["B"], "mean_ctx": acc["mean_ctx"], "launches": n, "dram_bytes_per_launch": dram / n,
                 "algorithmic_bytes_per_launch": acc["algorithmic_bytes"] / n,
                 "ratio": dram / acc["algorithmic_bytes"]})
    D += dram
    A += acc["algorithmic_bytes"]
    N += n
res = {"kernel": "decode_attn", "launches": N, "dram_bytes_per_launch": D / N, "algorithmic_bytes_per_launch": A / N,
       "ratio": D / A, "captures": caps,
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none over every "
                 "decode_attn launch of " + (src or "the captured runs") + " (engine path)"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
