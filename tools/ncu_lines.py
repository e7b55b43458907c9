"""Aggregate an ncu source page (SASS) by CUDA source line.

usage: ncu_lines.py <source.csv> <nvdisasm -g output> <metric column> [kernel index]
"""
import collections
import csv
import os
import re
import sys


def main():
    src_csv, sass, metric = sys.argv[1], sys.argv[2], sys.argv[3]
    kidx = int(sys.argv[4]) if len(sys.argv) > 4 else -1
    rows = list(csv.reader(open(src_csv)))
    blocks, cur = [], None
    for row in rows:
        if row and row[0] == "Kernel Name":
            cur = {"rows": []}
            blocks.append(cur)
            continue
        if row and row[0] == "Address":
            cur["hdr"] = row
            continue
        if cur is not None and "hdr" in cur:
            cur["rows"].append(row)
    addr2line, loc = {}, None
    for line in open(sass):
        if "## File" in line:
            m = re.search(r'File "([^"]+)", line (\d+)', line)
            if m:
                loc = (m.group(1), int(m.group(2)))
        m2 = re.search(r"/\*([0-9a-f]{4,5})\*/", line)
        if m2 and loc is not None:
            addr2line[int(m2.group(1), 16)] = loc
    b = blocks[kidx]
    h = b["hdr"]
    mi, ai = h.index(metric), h.index("Address")
    agg, tot, base = collections.Counter(), 0.0, None
    for row in b["rows"]:
        try:
            v = float(row[mi].replace(",", ""))
        except ValueError:
            continue
        a = int(row[ai], 16)
        base = a if base is None else base
        tot += v
        agg[addr2line.get(a - base, ("?", 0))] += v
    cache = {}
    for (f, ln), v in agg.most_common(30):
        if f not in cache:
            cache[f] = open(f).read().splitlines() if os.path.exists(f) else []
        txt = cache[f][ln - 1].strip()[:80] if 0 < ln <= len(cache[f]) else ""
        print(f"{v / tot * 100:5.1f}% {os.path.basename(f)}:{ln}: {txt}")


if __name__ == "__main__":
    main()
