"""Pivot attn_sweep_tc.py output: one row per (n, ctx), one column per (impl, split)."""
import json
import sys
from collections import defaultdict

for f in sys.argv[1:]:
    rows = [json.loads(l) for l in open(f) if l.startswith("{")]
    by = defaultdict(dict)
    cols = []
    for r in rows:
        c = (r["impl"], r["split"])
        if c not in cols:
            cols.append(c)
        by[(r["n"], r["ctx"])][c] = r["frac"]
    print(f)
    print("n,ctx".ljust(12) + "".join(f"{i}/{s}".rjust(8) for i, s in cols))
    for k, v in by.items():
        print(f"{k[0]},{k[1]}".ljust(12) + "".join((f"{v[c]:.3f}" if c in v else "-").rjust(8) for c in cols))
