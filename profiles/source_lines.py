#!/usr/bin/env python3
"""Top source lines of one kernel by warp-stall samples, from `ncu -i rep --page source --csv --print-source cuda,sass`.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python profiles/source_lines.py src.csv [top]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    hdr = next(r for r in rows if r and r[0] == "Line No")
    i_s, i_e = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    lines = []
    fname = ""
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
        if len(r) > i_e and r[0].isdigit() and r[2] == "-":        # per-line aggregate rows (no SASS address)
            lines.append((float(r[i_s] or 0), float(r[i_e] or 0), fname, int(r[0]), r[1].strip()))
    tot_s = sum(x[0] for x in lines) or 1.0
    tot_e = sum(x[1] for x in lines) or 1.0
    print(f"total warp-stall samples {tot_s:.0f}, warp instructions {tot_e:.0f}")
    print(" stall%   inst%   instructions  line")
    for s, e, f, ln, src in sorted(lines, key=lambda x: -x[0])[:top]:
        print(f"{100 * s / tot_s:6.1f}% {100 * e / tot_e:6.1f}% {e:14.0f}  {f}:{ln}: {src[:90]}")


if __name__ == "__main__":
    main()
