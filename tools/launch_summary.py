"""Sum an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name.

  python tools/launch_summary.py launches.csv
"""
import csv
import sys
from collections import defaultdict


def main(path):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0][:70]
        tot[name] += v
        cnt[name] += 1
    allv = sum(tot.values()) or 1.0
    for name, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v / 1e6:10.3f} ms  {100 * v / allv:5.1f}%  x{cnt[name]:<5d} {name}")


if __name__ == "__main__":
    main(sys.argv[1])
