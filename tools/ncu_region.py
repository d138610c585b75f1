"""Stall breakdown of a SASS region of an ncu report: the POTRF column loop (between the
first and the NB-th MUFU.RSQ64H of the first instantiation) or an address range."""
import csv
import subprocess
import sys

rep = sys.argv[1]
nmufu = int(sys.argv[2]) if len(sys.argv) > 2 else 16
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hdr, data = None, []
for r in csv.reader(out.splitlines()):
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
src = hdr.index("Source")
samp = hdr.index("Warp Stall Sampling (All Samples)")
ex = hdr.index("Instructions Executed")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
f = lambda x: float(x or 0)  # noqa: E731
mufu = [i for i, r in enumerate(data) if "MUFU.RSQ64H" in r[src]]
lo, hi = mufu[0] - 40, mufu[nmufu - 1] + 120
tot = {}
for r in data[lo:hi]:
    for i in st:
        tot[hdr[i]] = tot.get(hdr[i], 0) + f(r[i])
allsamp = sum(f(r[samp]) for r in data)
regsamp = sum(f(r[samp]) for r in data[lo:hi])
print(f"instructions in region {hi - lo}, samples {regsamp:.0f} of {allsamp:.0f}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]:
    print(f"  {k:24s} {v:8.0f}")
if len(sys.argv) > 3:
    for i in range(lo, hi):
        r = data[i]
        best = max(((f(r[j]), hdr[j][6:]) for j in st))
        print(f"{i:6d} {f(r[samp]):6.0f} {f(r[ex]):8.0f} {best[1]:12s} {r[src][:70]}")
