#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file F` launch list:
per kernel name, the number of launches and the median / last duration (us).

    python scripts/launch_times.py F [label]
"""
import collections
import csv
import statistics
import sys


def main():
    path = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else ""
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    t = collections.defaultdict(list)
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "ns")
            t[r["Kernel Name"].split("(")[0][:70]].append(v / 1000.0 if unit in ("nsecond", "ns") else v)
    for k, v in t.items():
        print(f"  {label:28s} {k:70s} n={len(v):3d} median={statistics.median(v):9.2f} us last={v[-1]:9.2f} us")


if __name__ == "__main__":
    main()
