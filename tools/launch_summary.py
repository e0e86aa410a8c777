"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch):
total and share per kernel name.  usage: launch_summary.py launches.csv"""
import collections
import csv
import sys


def main():
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    with open(sys.argv[1]) as f:
        rows = [r for r in csv.reader(line for line in f if not line.startswith("=="))]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    for r in rows[1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0][:70]
            v = float(r[vi].replace(",", ""))
            if v != v:  # a launch ncu could not time
                continue
            tot[name] += v
            cnt[name] += 1
    s = sum(tot.values())
    for name, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{v / 1e3:10.1f} us {100 * v / s:5.1f}% {cnt[name]:6d}x  {name}")


if __name__ == "__main__":
    main()
