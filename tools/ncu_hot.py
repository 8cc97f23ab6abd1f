"""Top SASS lines by warp-stall samples from an `ncu --page source --csv
--print-source sass` export (one or more kernels).
Usage: ncu_hot.py SOURCE.csv [N]"""
import csv
import sys


def main(path, n=25):
    lines = open(path).read().splitlines()
    kernels, cur = [], None
    i = 0
    while i < len(lines):
        if lines[i].startswith('"Kernel Name"'):
            cur = {"name": next(csv.reader([lines[i]]))[1], "rows": []}
            kernels.append(cur)
            hdr = next(csv.reader([lines[i + 1]]))
            cur["hdr"] = hdr
            i += 2
            continue
        if cur is not None and lines[i].strip():
            cur["rows"].append(next(csv.reader([lines[i]])))
        i += 1
    for k in kernels:
        h = k["hdr"]
        si = h.index("Warp Stall Sampling (All Samples)")
        src = h.index("Source")
        tot = sum(float(r[si] or 0) for r in k["rows"] if len(r) > si)
        print(f"== {k['name'][:100]}  total samples {tot:.0f}")
        top = sorted((r for r in k["rows"] if len(r) > si),
                     key=lambda r: -float(r[si] or 0))[:int(n)]
        for r in top:
            print(f"{float(r[si] or 0) / max(tot, 1):6.3f}  {r[0]:>6s}  {r[src][:90]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
