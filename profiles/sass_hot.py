#!/usr/bin/env python3
"""Top SASS instructions of an ncu source page (``ncu -i rep --page source --csv --print-source sass``):
per instruction the executed count and the stall samples, plus hot address ranges (loops).
Usage: sass_hot.py sass.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iA, iS, iSm, iI = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall = [(j, c) for j, c in enumerate(h) if c.startswith("stall_")]
recs = []
for r in rows[2:]:
    if len(r) <= iI:
        continue
    try:
        recs.append((int(r[iA], 16), r[iS].strip(), float(r[iSm] or 0), float(r[iI] or 0), {c: float(r[j] or 0) for j, c in stall}))
    except ValueError:
        pass
tot_s = sum(x[2] for x in recs); tot_i = sum(x[3] for x in recs)
print(f"samples {tot_s:.0f} instructions {tot_i:.0f}")
base = recs[0][0]
# consecutive windows of 32 instructions
win = {}
for a, s, sm, n, st in recs:
    k = (a - base) // (16 * 32)
    w = win.setdefault(k, [0, 0])
    w[0] += sm; w[1] += n
print("hot 32-instruction windows (offset: %samples %instructions):")
for k, (sm, n) in sorted(win.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"  0x{k*16*32:05x}: {100*sm/tot_s:5.1f}% smp {100*n/tot_i:5.1f}% ins")
