"""Aggregate an ncu source page (--print-source cuda,sass --csv) of the
search kernel by device function (line ranges of csrc/fph_search.cu).

usage: ncu_funcs.py <src.csv> [kernel index: 0 = first launch, 1 = second]
Prints executed warp instructions and stall samples per function, with the
top stall reasons of each.
"""
import collections
import csv
import re
import sys


def func_ranges(path):
    pat = re.compile(r"^(?:static )?(?:__device__|__global__|template)[^(]*?(\w+)\(")
    out = []
    for i, line in enumerate(open(path), 1):
        m = pat.match(line.strip()) if not line.startswith(" " * 8) else None
        if m and not line.lstrip().startswith("//"):
            out.append((i, m.group(1)))
    return out


def main():
    src, kidx = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1
    ranges = func_ranges("paper_2509_22432_b200/csrc/fph_search.cu")

    def fn(line):
        name = "?"
        for l, n in ranges:
            if line >= l:
                name = n
        return name

    rows = list(csv.reader(open(src)))
    sections, cur = [], None
    for r in rows:
        if r and r[0] == "File Path":
            cur = {"file": r[1].split("/")[-1], "rows": []}
            sections.append(cur)
            continue
        if r and r[0] == "Function Name":
            continue
        if r and r[0] == "Line No":
            cur["hdr"] = r
            continue
        if cur is not None and "hdr" in cur and r:
            cur["rows"].append(r)
    # sections repeat per kernel launch: split into halves by file order
    nfile = len({s["file"] for s in sections})
    per = len(sections) // max(1, len(sections) // nfile) if nfile else len(sections)
    launches = [sections[i:i + nfile] for i in range(0, len(sections), nfile)]
    secs = launches[kidx]
    inst = collections.Counter()
    stall = collections.defaultdict(collections.Counter)
    for s in secs:
        h = {k: i for i, k in enumerate(s["hdr"])}
        key = None
        for r in s["rows"]:
            if r[0] != "":
                ln = int(r[0])
                key = fn(ln) if s["file"] == "fph_search.cu" else s["file"]
                continue
            if r[2] == "...":
                continue
            try:
                inst[key] += float(r[h["Instructions Executed"]])
            except (ValueError, KeyError):
                pass
            for k, i in h.items():
                if k.startswith("stall_") and "Not Issued" not in k:
                    try:
                        stall[key][k[6:]] += float(r[i])
                    except ValueError:
                        pass
    ti = sum(inst.values())
    ts = sum(sum(c.values()) for c in stall.values())
    print(f"warp instructions {ti:.3e}, stall samples {ts:.0f}")
    for k, v in inst.most_common(25):
        ss = stall[k]
        tot = sum(ss.values())
        top = ", ".join(f"{n} {100 * x / max(tot, 1):.0f}%" for n, x in ss.most_common(3))
        print(f"{k:28s} inst {100 * v / ti:5.1f}%  samples {100 * tot / ts:5.1f}%  [{top}]")


if __name__ == "__main__":
    main()
