"""Summarise an ncu source page (CUDA+SASS view): stall samples per CUDA source line."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr = None
agg = defaultdict(lambda: [0.0, 0.0, ""])
cur = None
sass_top = []


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


for r in csv.reader(out.splitlines()):
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ii = hdr.index("Instructions Executed")
    if r[0] not in ("", "-"):
        cur = (r[0], r[1].strip()[:100])
    if r[2] in ("", "-"):
        continue
    key = cur if cur else ("?", "?")
    agg[key][0] += f(r[si])
    agg[key][1] += f(r[ii])
    sass_top.append((f(r[si]), r[3][:70], key[0] if key else "?"))
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"samples {tot:.0f}  instructions {toti:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/tot:5.1f}% smp {100*v[1]/toti:5.1f}% ins  L{k[0]:>5} {k[1]}")
print("--- top SASS ---")
for s in sorted(sass_top, reverse=True)[:15]:
    print(f"{100*s[0]/tot:5.1f}%  L{s[2]}  {s[1]}")
