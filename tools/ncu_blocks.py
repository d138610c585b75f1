"""Per-block (100 SASS instructions) sample / stall summary of an ncu source page export."""
import csv
import sys

path = sys.argv[1]
step = int(sys.argv[2]) if len(sys.argv) > 2 else 100
hdr, data = None, []
for r in csv.reader(open(path).read().splitlines()):
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
total = sum(f(r[samp]) for r in data)
print(f"total samples {total:.0f}")
for a in range(0, len(data), step):
    b = min(a + step, len(data))
    sm = sum(f(r[samp]) for r in data[a:b])
    if sm < 0.005 * total:
        continue
    tot = {}
    kinds = {}
    for r in data[a:b]:
        for i in st:
            tot[hdr[i][6:]] = tot.get(hdr[i][6:], 0) + f(r[i])
        w = r[src].split()
        op = (w[1] if w and w[0].startswith("@") and len(w) > 1 else (w[0] if w else "")).split(".")[0]
        kinds[op] = kinds.get(op, 0) + 1
    top = ", ".join(f"{k} {v / sm * 100:.0f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:3])
    ks = " ".join(f"{k}:{v}" for k, v in sorted(kinds.items(), key=lambda kv: -kv[1])[:5])
    print(f"{a:5d}-{b:5d} {sm / total * 100:5.1f}%  [{top}]  {ks}")
