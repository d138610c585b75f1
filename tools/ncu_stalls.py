"""Stall-reason breakdown for a CUDA source line range of an ncu report (source page)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
fname = sys.argv[4] if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr = None
cur = None
tot = defaultdict(float)
for r in csv.reader(out.splitlines()):
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0] not in ("", "-"):
        cur = int(r[0]) if r[0].isdigit() else None
        continue
    if cur is None or not (lo <= cur <= hi):
        continue
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                tot[h] += float(r[i])
            except ValueError:
                pass
s = sum(tot.values()) or 1
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v:
        print(f"{k:28s} {v:8.0f} {100*v/s:5.1f}%")
