#!/usr/bin/env python
"""Hottest SASS instructions (warp-stall samples) of an .ncu-rep, with the
source line they map to:  python scripts/ncu_hot.py rep.ncu-rep [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                      text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = [(int(r[iss] or 0), r[ia], r[isrc].strip()) for r in rows[2:] if len(r) > iss]
tot = sum(d[0] for d in data) or 1
for s, a, src in sorted(data, reverse=True)[:top]:
    print(f"{100.0 * s / tot:5.1f}%  {a[-5:]}  {src}")
