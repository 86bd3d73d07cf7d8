"""Per-source-line warp-stall samples of an ncu report (--page source,
cuda,sass interleaved): the top lines and the stall-reason totals.
usage: python scripts/ncu_lines.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = None
hdr = None
lines = []
tot = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    ix = {h: i for i, h in enumerate(hdr)}
    samp = r[ix["# Samples"]]
    samp = int(samp) if samp.isdigit() else 0
    if samp:
        lines.append((samp, cur, int(r[0]), r[1].strip()[:80]))
    for h, i in ix.items():
        if h.startswith("stall_") and i < len(r):
            try:
                tot[h] = tot.get(h, 0) + float(r[i] or 0)
            except ValueError:
                pass
lines.sort(reverse=True)
for l in lines[:top]:
    print(l)
print(sorted(((round(v), k) for k, v in tot.items() if v), reverse=True)[:12])
