#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file X): per kernel
name, launch count, average duration and share of the total.  Usage: launch_summary.py launches.csv"""
import collections
import csv
import sys


def main(path, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        tot[r[ik]] += v
        cnt[r[ik]] += 1
    all_t = sum(tot.values()) or 1.0
    print(title)
    print("cold-cache, serialised launches: compare SHARES, not absolutes")
    for k, v in tot.most_common():
        print(f"{100 * v / all_t:6.2f}%  {cnt[k]:4d} launches  avg {v / cnt[k] / 1e3:8.2f} us  {k[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
