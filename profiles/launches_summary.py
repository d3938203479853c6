#!/usr/bin/env python3
"""Per-kernel launch counts, mean duration and share of the summed device time, from an ncu launch list

    ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file launches.csv python bench.py ...
    python profiles/launches_summary.py launches.csv "<command line, for the header>"

ncu serialises and cold-starts every launch, so the shares are meaningful and the absolute times are not.
"""
import collections
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if r]
    hdr = next(r for r in rows if "Kernel Name" in r and "Metric Value" in r)
    i_k, i_m, i_v, i_u, i_id = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                                hdr.index("Metric Unit"), hdr.index("ID"))
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
    per = collections.defaultdict(list)
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) > i_v and r[i_m] == "gpu__time_duration.sum":
            name = r[i_k].split("(")[0][:70]
            per[name].append(float(r[i_v].replace(",", "")) * scale.get(r[i_u], 1.0))
    total = sum(sum(v) for v in per.values()) or 1.0
    if len(sys.argv) > 2:
        print(sys.argv[2])
    print(f"{'kernel':70s} {'launches':>9s} {'mean_us':>10s} {'share':>7s}")
    for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{name:70s} {len(v):9d} {sum(v) / len(v):10.1f} {100 * sum(v) / total:6.1f}%")


if __name__ == "__main__":
    main()
