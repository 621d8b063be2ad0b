"""Stall-reason breakdown from an ncu report's source page (needs -lineinfo, --import-source).

usage: python tools/ncu_stalls.py REPORT [TOP]   -> kernel-wide stall totals, then the top
CUDA source lines with their dominant stall reasons.
"""
import csv, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, cur, per_line, tot = None, None, defaultdict(lambda: defaultdict(float)), defaultdict(float)
src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Name" or r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if not hdr or len(r) != len(hdr):
        continue
    key = (cur, r[0]); src[key] = r[1]
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                v = float(r[i] or 0)
            except ValueError:
                continue
            per_line[key][h] += v; tot[h] += v
allv = sum(tot.values()) or 1
print("kernel stall totals:", ", ".join(f"{k[6:]} {100*v/allv:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
ranked = sorted(per_line.items(), key=lambda kv: -sum(kv[1].values()))[:top]
for (f, ln), d in ranked:
    s = sum(d.values())
    tops = ", ".join(f"{k[6:]} {100*v/s:.0f}%" for k, v in sorted(d.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{100*s/allv:5.1f}% {f}:{ln:>5} [{tops}] {src[(f, ln)].strip()[:80]}")
