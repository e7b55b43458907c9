"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch):
per kernel name, launches and total microseconds, in launch order.

  python tools/launch_table.py gpurun_out/launches.csv
"""

import csv
import re
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    order, agg = [], {}
    for r in data:
        name = re.sub(r"\(.*", "", r[ki]).replace("fph::<unnamed>::", "")[:70]
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        if name not in agg:
            order.append(name)
            agg[name] = [0, 0.0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v for _, v in agg.values())
    for name in order:
        n, v = agg[name]
        print(f"{v:10.1f} us  x{n:<3d} {name}")
    print(f"{tot:10.1f} us  total ({len(data)} launches)")


if __name__ == "__main__":
    main(sys.argv[1])
