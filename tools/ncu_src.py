"""Summarise an ncu source page (CUDA view): top lines by stall samples and instructions."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows, fname, header = [], None, None
for rec in csv.reader(out.splitlines()):
    if not rec:
        continue
    if rec[0] == "File Name":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        header = rec
        continue
    if header is None or len(rec) != len(header):
        continue
    d = dict(zip(header, rec))
    try:
        samp = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst = float(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    rows.append((samp, inst, fname, d["Line No"], d["Source"].strip()[:110]))
tot_s = sum(r[0] for r in rows) or 1
tot_i = sum(r[1] for r in rows) or 1
print(f"total samples {tot_s:.0f}, instructions {tot_i:.0f}")
for r in sorted(rows, reverse=True)[:top]:
    print(f"{100*r[0]/tot_s:5.1f}% smp {100*r[1]/tot_i:5.1f}% ins  {r[2]}:{r[3]}  {r[4]}")
