"""DRAM traffic vs algorithmic bytes over windows of one job's launches of a
kernel class (ncu -s SKIP -c COUNT captures of scripts/traffic_job.py runs),
matched launch by launch with the engine's per-launch algorithmic bytes
(gpurun_out/traffic_job_<class>_bytes.npy) -> profiles/rN/traffic_<class>.json,
read by bench.py for roofline.traffic.

    python scripts/traffic_windows.py OUT.json SKIP:CSV [SKIP:CSV ...]"""
import csv
import json
import os
import sys

import numpy as np


def per_launch(path, cls):
    rows = list(csv.reader(open(path)))
    hdr, byid = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if cls in d["Kernel Name"] and d["Metric Name"].startswith("dram__bytes"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d.get("Metric Unit", "byte"), 1)
                byid[int(d["ID"])] = byid.get(int(d["ID"]), 0.0) + float(d["Metric Value"].replace(",", "")) * scale
    return [byid[i] for i in sorted(byid)]


out, args = sys.argv[1], sys.argv[2:]
cls = "decode_attn"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
alg = np.load(os.path.join(root, "gpurun_out", f"traffic_job_{cls}_bytes.npy"))
wins, D, A = [], 0.0, 0.0
for a in args:
    skip, path = a.split(":", 1)
    skip = int(skip)
    dram = per_launch(path, cls)
    n = len(dram)
    al = alg[skip:skip + n]
    wins.append({"skip": skip, "launches": n, "dram_bytes_per_launch": sum(dram) / n,
                 "algorithmic_bytes_per_launch": float(al.sum()) / n, "ratio": sum(dram) / float(al.sum())})
    D += sum(dram)
    A += float(al.sum())
N = sum(w["launches"] for w in wins)
res = {"kernel": cls, "launches": N, "job_launches": int(len(alg)), "dram_bytes_per_launch": D / N,
       "algorithmic_bytes_per_launch": A / N, "ratio": D / A, "windows": wins,
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none over windows of the "
                 "decode_attn launches of ONE C2 bench job (scripts/traffic_job.py: 256 requests, 32 layers), each "
                 "launch matched with the engine's algorithmic bytes of the same launch"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
