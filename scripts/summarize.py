"""Summarise gpurun_out: bench line + ncu launch lists."""
import collections
import csv
import json
import sys

def bench(path):
    l = [x for x in open(path) if x.startswith('{')]
    if not l:
        print(open(path).read()[-1500:]); return
    d = json.loads(l[0])
    for k in ['value', 'ms_per_step', 'bubble_pct', 'gpu_launches', 'e2e', 'roofline']:
        print(k, d.get(k))
    for k, v in d.get('kernels', {}).items():
        print(f"  {k:16s} {v['ms']:9.1f} ms {v['GB/s']:8.1f} GB/s {v['TFLOP/s']:7.1f} TF  n={v['launches']}")

def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None; data = []
    for r in rows:
        if r and r[0] == 'ID': hdr = r; continue
        if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in data:
        agg[r['Kernel Name'][:55]][r['Metric Name']].append(float(r['Metric Value'].replace(',', '')))
    print(path)
    for k, v in agg.items():
        t = v.get('gpu__time_duration.sum', [0]); rd = v.get('dram__bytes_read.sum', [0]); wr = v.get('dram__bytes_write.sum', [0])
        n = len(t)
        print(f"  {k:55s} n={n:3d} t={sum(t)/n/1e3:8.2f}us rd={sum(rd)/n/1e6:8.2f}MB wr={sum(wr)/n/1e6:7.2f}MB GB/s={(sum(rd)+sum(wr))/max(sum(t),1):7.1f}")

for p in sys.argv[1:]:
    (bench if p.endswith('.log') else launches)(p)
