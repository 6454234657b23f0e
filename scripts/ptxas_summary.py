#!/usr/bin/env python
"""Registers / stack / spills per kernel from an nvcc -Xptxas -v log."""
import re, sys
info = {}
cur_regs = None
cur_props = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur_regs = m.group(1); info.setdefault(cur_regs, {})
        continue
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur_props = m.group(1); info.setdefault(cur_props, {})
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
    if m and cur_props:
        info[cur_props]["stack"] = int(m.group(1)); info[cur_props]["spill"] = int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur_regs:
        info[cur_regs]["regs"] = int(m.group(1))
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for n, r in info.items():
    m = re.search(r"k_fft_persistI(.)Li(\d+)ELi(\d+)ELi(\d+)ELi(\d)ELi(\d+)E", n)
    if m:
        n = f"persist {'c64' if m.group(1)=='f' else 'c128'} P={m.group(2)} NT={m.group(3)} TPB={m.group(4)} {'chirp' if m.group(5)=='1' else 'afft'} MINB={m.group(6)}"
    if flt in n and "regs" in r:
        print(f"{n:70s} regs={r.get('regs')} stack={r.get('stack',0)} spill={r.get('spill',0)}")
