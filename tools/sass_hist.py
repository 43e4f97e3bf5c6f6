"""Per-opcode executed-instruction histogram from `ncu -i rep --page source --csv --print-source sass`.

python tools/sass_hist.py src.csv UNITS  -> instructions per unit (e.g. per token), by opcode and by region
"""
import collections
import csv
import re
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    hdr = rows[1]
    ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    ops = collections.Counter()
    samp = collections.Counter()
    tot = 0
    seq = []
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        n = float(r[iex] or 0)
        src = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip())
        op = src.split()[0].split(".")[0] if src else "?"
        ops[op] += n
        samp[op] += float(r[isamp] or 0)
        tot += n
        seq.append((r[ia], n, int(float(r[isamp] or 0)), r[isrc].strip()))
    print(f"total {tot / units:.1f} per unit")
    for op, n in ops.most_common(45):
        print(f"{op:10s} {n / units:8.1f}  stall-samples {int(samp[op])}")
    if len(sys.argv) > 3:
        for a, n, s, src in seq:
            if n / units >= float(sys.argv[3]):
                print(f"{a[-5:]} {n / units:6.2f} {s:6d} {src}")


if __name__ == "__main__":
    main()
