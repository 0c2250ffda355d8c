"""Stall-reason breakdown of an ncu report by SASS address region.
    python tools/ncu_regions.py rep.ncu-rep [split_index ...]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
splits = [int(a) for a in sys.argv[2:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(out.splitlines()))
h, rows = r[1], r[2:]
st = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
bounds = [0] + splits + [len(rows)]
for a, b in zip(bounds, bounds[1:]):
    tot = {h[i]: sum(int(x[i] or 0) for x in rows[a:b]) for i in st}
    s = sum(tot.values())
    top = sorted(tot.items(), key=lambda kv: -kv[1])[:7]
    print(f"[{a},{b}) samples {s}: " + ", ".join(f"{k[6:]} {v}" for k, v in top))
