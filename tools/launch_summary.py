"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum) into
per-kernel counts, total ms and share of device time.
Usage: launch_summary.py LAUNCHES.csv OUT.txt "header line" """
import collections
import csv
import re
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0}


def short(name):
    n = name.replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    n = re.sub(r"^void ", "", n)
    depth, out = 0, ""
    for ch in n:  # drop template arguments
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif depth == 0:
            out += ch
    return out.split("(")[0].split("::")[-1]


def main(src, dst, header):
    rows = list(csv.reader(open(src)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = (h.index("Kernel Name"), h.index("Metric Value"),
                  h.index("Metric Unit"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-6)
        k = short(r[ki])
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(x[1] for x in agg.values())
    out = [header, f"total device time {tot:.3f} ms over "
           f"{sum(x[0] for x in agg.values())} launches",
           f"{'kernel':40s} {'n':>5s} {'ms':>10s} {'share':>6s}"]
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:40s} {n:5d} {ms:10.3f} {ms / tot:6.3f}")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out[:30]))


if __name__ == "__main__":
    main(*sys.argv[1:4])
